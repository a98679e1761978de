// Host-visible kernel registry: type-erased launchers for every compiled
// (dtype, degree bucket, checks-per-thread, variable-degree bucket) variant.
#pragma once

#include <cuda_runtime.h>
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <stdint.h>

#include "resident.cuh"
#include "resident_regular.cuh"
#include "streaming.cuh"
#include "sharded.cuh"
#include "wide.cuh"

namespace admm {

struct ResidentGraphArgs {
  int n_vars, n_checks, m_pad;
  const int* chk_var;
  const uint16_t* var_pos;
  const uint8_t* var_deg;
  const int* edge_base;
  const int* var_edge;  // [n_vars][DV] reference edge ids (regular kernels)
  const int* var_orig;  // relabeled regular layout (layout.h), may be null
  const int* edge_ref;
  const int* var_edge_int;  // relabeled: [internal var][DV] internal edge c*D + k
  const int* check_rot;     // colored layout rotations (null = none)
};

struct ResidentFrameArgs {
  long long batch;
  const void* gamma;
  long long ld_gamma;
  double mu, rho, thr;
  int t_max;
  const void* z_in;
  const void* lam_in;
  long long ld_edge;
  void* x_out;
  long long ld_x;
  uint8_t* hard_out;
  long long ld_hard;
  int* iters_out;
  uint8_t* flags_out;
  int* weight_out;
  void* z_out;
  void* lam_out;
  int* queue;
  SynthParams synth;
};

using ResidentLaunchFn = cudaError_t (*)(const ResidentGraphArgs&, const ResidentFrameArgs&, int grid, int nt,
                                         int smem, cudaStream_t st);

struct ResidentLaunch {
  const void* fn;
  ResidentLaunchFn launch;
  int smem, occupancy, regs;
  bool colored;  // regular kernel on the colored message layout (layout.h)
  int np_fixed;  // compile-time padded variable count (0 = computed from n_vars)
  bool gm_smem;  // LLR steps in shared memory (regular_gm_smem)
  int zs_cpt;    // > 0: edge state in shared memory for this many checks per thread
};

// The stop-rule threshold in T, rounded toward +inf: a partial sum >= it is
// >= the fp64 threshold (early-out tests stay exact in fp32 mode).
template <typename T>
inline T thr_round_up(double thr) {
  if constexpr (sizeof(T) == 8) {
    return thr;
  } else {
    float f = static_cast<float>(thr);
    if (static_cast<double>(f) < thr) f = std::nextafter(f, INFINITY);
    return f;
  }
}

// Fixed-point scale of the fp32 stop-rule sums (ResidentParams::fx_scale):
// the power of two that puts the fp32 threshold in [2^20, 2^21).
inline float fx_scale_of(double thr) {
  int e;
  std::frexp(static_cast<double>(thr_round_up<float>(thr)), &e);  // thr_f = m 2^e, m in [0.5, 1)
  return std::ldexp(1.0f, 21 - e);
}
inline unsigned long long fx_thr_of(double thr) {
  return static_cast<unsigned long long>(std::ceil(thr * static_cast<double>(fx_scale_of(thr)) * 2097152.0));
}

template <typename T>
ResidentParams<T> make_params(const ResidentGraphArgs& g, const ResidentFrameArgs& a) {
  ResidentParams<T> p;
  p.n_vars = g.n_vars;
  p.n_checks = g.n_checks;
  p.m_pad = g.m_pad;
  p.chk_var = g.chk_var;
  p.var_pos = g.var_pos;
  p.var_deg = g.var_deg;
  p.edge_base = g.edge_base;
  p.var_orig = g.var_orig;
  p.edge_ref = g.edge_ref;
  p.check_rot = g.check_rot;
  p.batch = a.batch;
  p.gamma = static_cast<const T*>(a.gamma);
  p.ld_gamma = a.ld_gamma;
  p.mu = T(a.mu);
  p.inv_mu = T(1.0 / a.mu);
  p.rho = T(a.rho);
  p.one_minus_rho = T(1.0 - a.rho);
  p.thr = thr_round_up<T>(a.thr);
  p.thr_d = a.thr;
  p.fx_scale = fx_scale_of(a.thr);
  p.fx_thr = fx_thr_of(a.thr);
  p.t_max = a.t_max;
  p.z_in = static_cast<const T*>(a.z_in);
  p.lam_in = static_cast<const T*>(a.lam_in);
  p.ld_edge = a.ld_edge;
  p.x_out = static_cast<T*>(a.x_out);
  p.ld_x = a.ld_x;
  p.hard_out = a.hard_out;
  p.ld_hard = a.ld_hard;
  p.iters_out = a.iters_out;
  p.flags_out = a.flags_out;
  p.weight_out = a.weight_out;
  p.z_out = static_cast<T*>(a.z_out);
  p.lam_out = static_cast<T*>(a.lam_out);
  p.queue = a.queue;
  p.synth = a.synth;
  return p;
}

template <typename T, int D, int CPT, int DVMAX>
cudaError_t launch_resident(const ResidentGraphArgs& g, const ResidentFrameArgs& a, int grid, int nt, int smem,
                            cudaStream_t st) {
  resident_decode_kernel<T, D, CPT, DVMAX><<<grid, nt, smem, st>>>(make_params<T>(g, a));
  return cudaGetLastError();
}

template <typename T, int D, int DV, int CPT, int VPT, int MINB, int MAXT, bool COL, int NPC, int NTC, bool ZS>
cudaError_t launch_regular(const ResidentGraphArgs& g, const ResidentFrameArgs& a, int grid, int nt, int smem,
                           cudaStream_t st) {
  resident_regular_kernel<T, D, DV, CPT, VPT, MINB, MAXT, COL, NPC, NTC, ZS><<<grid, nt, smem, st>>>(
      make_params<T>(g, a), g.var_edge_int ? g.var_edge_int : g.var_edge);
  return cudaGetLastError();
}

// Regular-code variants: (D, DV, CPT, VPT).  `variant` enumerates the
// compiled shapes that match; returns false past the last one.
bool regular_lookup_f32(int D, int DV, int CPT, int VPT_min, int nt, int n_vars, int variant, int* VPT,
                        ResidentLaunch* out);
bool regular_lookup_f64(int D, int DV, int CPT, int VPT_min, int nt, int n_vars, int variant, int* VPT,
                        ResidentLaunch* out);
inline bool regular_lookup(int dtype, int D, int DV, int CPT, int VPT_min, int nt, int n_vars, int variant,
                           int* VPT, ResidentLaunch* out) {
  return dtype ? regular_lookup_f64(D, DV, CPT, VPT_min, nt, n_vars, variant, VPT, out)
               : regular_lookup_f32(D, DV, CPT, VPT_min, nt, n_vars, variant, VPT, out);
}

// Defined in resident_f32.cu / resident_f64.cu.
bool resident_lookup_f32(int D, int CPT, int DVMAX, ResidentLaunch* out);
bool resident_lookup_f64(int D, int CPT, int DVMAX, ResidentLaunch* out);
inline bool resident_lookup(int dtype, int D, int CPT, int DVMAX, ResidentLaunch* out) {
  return dtype ? resident_lookup_f64(D, CPT, DVMAX, out) : resident_lookup_f32(D, CPT, DVMAX, out);
}

// ---- streaming engine ----
struct StreamGraphArgs {
  int n_vars, n_checks, n_edges, m_pad, dvmax;
  const int* chk_var;
  const int* edge_base;
  const int* var_edge;
  const int* ctbl = nullptr;  // wide engine index tables
  const int* vtbl = nullptr;
};

struct StreamLaunch {
  const void* fn;
  int (*launch)(const StreamGraphArgs&, const ResidentFrameArgs&, int S, void* ws, int grid, cudaStream_t st);
  int occupancy, regs;
};

template <typename T>
StreamParams<T> make_stream_params(const StreamGraphArgs& g, const ResidentFrameArgs& a, int S, void* ws,
                                   long long ncblk, bool sharded) {
  StreamParams<T> p{};
  p.n_vars = g.n_vars;
  p.n_checks = g.n_checks;
  p.n_edges = g.n_edges;
  p.m_pad = g.m_pad;
  p.chk_var = g.chk_var;
  p.edge_base = g.edge_base;
  p.var_edge = g.var_edge;
  p.dvmax = g.dvmax;
  p.batch = a.batch;
  p.gamma = static_cast<const T*>(a.gamma);
  p.ld_gamma = a.ld_gamma;
  p.mu = T(a.mu);
  p.inv_mu = T(1.0 / a.mu);
  p.rho = T(a.rho);
  p.one_minus_rho = T(1.0 - a.rho);
  p.thr = thr_round_up<T>(a.thr);
  p.thr_d = a.thr;
  p.t_max = a.t_max;
  p.x_out = static_cast<T*>(a.x_out);
  p.ld_x = a.ld_x;
  p.hard_out = a.hard_out;
  p.ld_hard = a.ld_hard;
  p.iters_out = a.iters_out;
  p.flags_out = a.flags_out;
  p.weight_out = a.weight_out;
  p.S = S;
  p.synth = a.synth;
  const StreamLayout L(sizeof(T), g.n_edges, g.n_vars, ncblk, S, sharded);
  char* base = static_cast<char*>(ws);
  p.zl = reinterpret_cast<T*>(base + L.zl);
  p.msg = reinterpret_cast<T*>(base + L.msg);
  p.x = reinterpret_cast<T*>(base + L.x);
  p.gm = reinterpret_cast<T*>(base + L.gm);
  p.part = reinterpret_cast<T*>(base + L.part);
  p.frame = reinterpret_cast<long long*>(base + L.ints);
  int* ib = reinterpret_cast<int*>(base + L.ints + StreamLayout::al(sizeof(long long) * S));
  p.notconv = ib;
  p.st = ib + S;
  p.tcount = ib + 2 * S;
  p.conv = ib + 3 * S;
  p.weight = ib + 4 * S;
  p.nonint = ib + 5 * S;
  p.odd = ib + 6 * S;
  p.ctr = ib + 7 * S;
  p.flagpad = reinterpret_cast<int*>(base + L.flags);
  return p;
}

template <typename T, int D, int DVMAX, bool REG>
int launch_streaming(const StreamGraphArgs& g, const ResidentFrameArgs& a, int S, void* ws, int grid,
                     cudaStream_t st) {
  StreamParams<T> p = make_stream_params<T>(g, a, S, ws, (g.n_checks + kStreamCK - 1) / kStreamCK, false);
  void* args[] = {&p};
  return (int)cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(&streaming_decode_kernel<T, D, DVMAX, REG>),
                                          grid, kStreamThreads, args, 0, st);
}

struct ShardLaunch {
  const void* fn;
  int (*launch)(const StreamGraphArgs&, const ResidentFrameArgs&, int S, void* ws, int grid, const ShardGeom& geo,
                cudaStream_t st);
};

template <typename T, int D, int DVMAX, bool REG>
int launch_sharded(const StreamGraphArgs& g, const ResidentFrameArgs& a, int S, void* ws, int grid,
                   const ShardGeom& geo, cudaStream_t st) {
  StreamParams<T> p = make_stream_params<T>(g, a, S, ws, grid, true);
  ShardGeom gg = geo;
  void* args[] = {&p, &gg};
  return (int)cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(&sharded_decode_kernel<T, D, DVMAX, REG>),
                                          grid, ShardThreads<T>::value, args, geo.total, st);
}

bool shard_lookup(int dtype, int D, int DVMAX, bool regular, ShardLaunch* out);
bool phase_profile(int enable, unsigned long long* out8);

bool stream_lookup(int dtype, int D, int DVMAX, bool regular, StreamLaunch* out);

// Defined in project.cu.
bool launch_project(int dtype, int D, long long m, int d, const void* in, void* out, cudaStream_t st);
void launch_synth(int dtype, long long batch, int n, const SynthParams& s, void* out, long long ld, cudaStream_t st);


// ---- wide streaming engine (wide.cuh) ----
struct WideLaunch {
  const void* fn;
  int (*launch)(const StreamGraphArgs&, const ResidentFrameArgs&, int S, void* ws, int grid, cudaStream_t st);
  int occupancy, regs, vs, smem, D, DV;
};

inline long long wide_ncb(int n_checks) { return (n_checks + kWideCB - 1) / kWideCB; }

template <typename T>
WideParams<T> make_wide_params(const StreamGraphArgs& g, const ResidentFrameArgs& a, int S, void* ws) {
  WideParams<T> p{};
  p.n_vars = g.n_vars;
  p.n_checks = g.n_checks;
  p.n_edges = g.n_edges;
  p.m_pad = g.m_pad;
  p.dvmax = g.dvmax;
  p.chk_var = g.chk_var;
  p.edge_base = g.edge_base;
  p.var_edge = g.var_edge;
  p.ctbl = g.ctbl;
  p.vtbl = g.vtbl;
  p.batch = a.batch;
  p.gamma = static_cast<const T*>(a.gamma);
  p.ld_gamma = a.ld_gamma;
  p.mu = T(a.mu);
  p.rho = T(a.rho);
  p.one_minus_rho = T(1.0 - a.rho);
  p.thr = thr_round_up<T>(a.thr);
  p.thr_d = a.thr;
  p.t_max = a.t_max;
  p.x_out = static_cast<T*>(a.x_out);
  p.ld_x = a.ld_x;
  p.hard_out = a.hard_out;
  p.ld_hard = a.ld_hard;
  p.iters_out = a.iters_out;
  p.flags_out = a.flags_out;
  p.weight_out = a.weight_out;
  p.S = S;
  p.ncb = static_cast<int>(wide_ncb(g.n_checks));

  p.synth = a.synth;
  const WideLayout L(sizeof(T), g.n_edges, g.n_vars, p.ncb, S, a.synth.kind != 0);
  char* base = static_cast<char*>(ws);
  p.zl = reinterpret_cast<T*>(base + L.zl);
  p.msg = reinterpret_cast<T*>(base + L.msg);
  p.x = reinterpret_cast<T*>(base + L.x);
  p.gm = reinterpret_cast<T*>(base + L.gm);
  p.part = reinterpret_cast<T*>(base + L.part);
  p.gfr = a.synth.kind != 0 ? reinterpret_cast<T*>(base + L.gfr) : nullptr;
  p.vpart = reinterpret_cast<int*>(base + L.vpart);
  p.direct = (a.x_out == nullptr && a.hard_out == nullptr && std::getenv("ADMM_B200_WIDE_RETIRE_PASS") == nullptr) ? 1 : 0;
  int* ib = reinterpret_cast<int*>(base + L.ints);
  p.st = ib;
  p.tcount = ib + S;
  p.conv = ib + 2 * S;
  p.weight = ib + 3 * S;
  p.nonint = ib + 4 * S;
  p.odd = ib + 5 * S;
  p.frame = ib + 6 * S;
  p.fnext = ib + 7 * S;
  p.slist = ib + 8 * S;  // two lists of S
  p.ctr = ib + 10 * S;
  return p;
}

template <typename T, int VS, int D, int DVMAX, bool REG, int NS, int MINB>
int launch_wide(const StreamGraphArgs& g, const ResidentFrameArgs& a, int S, void* ws, int grid, cudaStream_t st) {
  WideParams<T> p = make_wide_params<T>(g, a, S, ws);
  void* args[] = {&p};
  return (int)cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(&wide_decode_kernel<T, VS, D, DVMAX, REG, NS, MINB>),
                                          grid, kWideThreads, args, wide_smem_bytes<T, VS, D, DVMAX, NS>(), st);
}

// Defined in wide.cu.
bool wide_lookup(int dtype, int D, int DVMAX, bool regular, WideLaunch* out);
bool wide_phase_profile(int enable, unsigned long long* out8);

}  // namespace admm
