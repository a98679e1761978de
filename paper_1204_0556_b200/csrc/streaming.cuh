// Streaming engine: codes too large for one SM (BASELINE config 5, n = 16384).
//
// State is batch-interleaved over S frame SLOTS (S a multiple of 32): every
// edge row holds the S slots' values contiguously, so a warp -- 32 slots of
// ONE check or ONE variable -- reads and writes 128 B (fp32) / 256 B (z,lambda
// pairs) per access with warp-uniform graph indices:
//     zl  [E][S] (z, lambda) pairs    msg [E][S] z - lambda/mu
//     x   [N][S]                      gm  [N][S] gamma/mu
// S is sized so the whole state stays resident in the 126 MB L2.
//
// One cooperative persistent kernel runs every iteration of every slot; grid
// syncs separate three phases (reference admm_decoder.py:171-181):
//   V  variable update  x = clip((sum msg - gamma/mu)/deg)          (:108-124)
//   C  check update     fused z-update, projection, residual partials,
//                       lambda-update, message write                (:127-149)
//   S  slot management  stop rule (:169,179), retirement, refill
// A slot's life: FRESH (new frame, z = lambda = 0 implicit) -> RUNNING ->
// RETIRING (converged or t_max: the next V/C pass only computes its output
// statistics from the final x) -> next frame or EMPTY.  Retirement is per
// slot, so heavy-tailed iteration counts never hold converged frames.
//
// The stop rule uses the same exact shortcut as the resident engine: a check
// tile whose partial residual already reaches eps^2*E sets the slot's
// not-converged flag; only slots with no flag sum their partials (one warp,
// fixed tree -> deterministic).
#pragma once

#include <cooperative_groups.h>

#include "common.cuh"
#include "projection.cuh"
#include "synth.cuh"

namespace admm {

enum : int { kSlotEmpty = 0, kSlotFresh = 1, kSlotRunning = 2, kSlotRetiring = 3 };

constexpr int kStreamCK = 8;   // checks per phase-C tile (one warp each)
constexpr int kStreamVK = 8;   // variables per phase-V tile (one warp each)
constexpr int kStreamThreads = 256;

template <typename T>
struct StreamParams {
  // graph
  int n_vars, n_checks, n_edges, m_pad;
  const int* chk_var;    // [Dbucket][m_pad], -1 = unused slot
  const int* edge_base;  // [n_checks] reference edge id of slot 0
  const int* var_edge;   // [n_vars][dvmax] reference edge ids, -1 = unused
  int dvmax;
  // frames
  long long batch;
  const T* gamma;
  long long ld_gamma;
  T mu, inv_mu, rho, one_minus_rho, thr;  // thr: eps^2 E rounded up to T (early-out tests)
  double thr_d;                            // eps^2 E: the exact sums are fp64
  int t_max;
  // outputs
  T* x_out;
  long long ld_x;
  uint8_t* hard_out;
  long long ld_hard;
  int* iters_out;
  uint8_t* flags_out;
  int* weight_out;
  // workspace
  int S;
  T* zl;              // [E][S][2]
  T* msg;             // [E][S]
  T* x;               // [N][S]
  T* gm;              // [N][S]
  T* part;            // [n_cblk][S][2]
  int* notconv;       // [S]
  int* st;            // [S] slot state
  int* tcount;        // [S] iterations run
  long long* frame;   // [S]
  int* conv;          // [S] converged flag of a retiring slot
  int* weight;        // [S] hard-decision weight (retiring)
  int* nonint;        // [S] non-integral flag (retiring)
  int* odd;           // [S] odd-parity flag (retiring)
  int* ctr;           // [0] queue, [1] active slots, [2] passes
  SynthParams synth;  // fused frame synthesis (kind 0 = read gamma)
  int* flagpad;       // [4][S][32] not-converged flags, one cache line per slot (sharded engines)
};

// Bytes of streaming workspace for S slots.
struct StreamLayout {
  size_t zl, msg, x, gm, part, ints, flags, total;
  static size_t al(size_t b) { return (b + 255) & ~size_t(255); }
  StreamLayout(size_t elem, long long E, long long N, long long ncblk, long long S, bool sharded = false) {
    size_t o = 0;
    zl = o; o += sharded ? 0 : al(elem * 2 * E * S);  // sharded: z, lambda live in shared memory
    msg = o; o += al(elem * E * S);
    x = o; o += al(elem * N * S);
    gm = o; o += sharded ? 0 : al(elem * N * S);
    part = o; o += al(elem * 2 * ncblk * S);
    ints = o; o += al(sizeof(long long) * S) + al(sizeof(int) * (7 * S + 8));
    flags = o; o += al(sizeof(int) * 4 * 32 * S);  // per-slot flags, one 128-byte line each
    total = o;
  }
};

template <typename T, int D, int DVMAX>
__device__ __forceinline__ void stream_phase_v(const StreamParams<T>& p, int tile, int n_vtiles_x, int* sred) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int i = (tile % n_vtiles_x) * kStreamVK + w;
  const int s = (tile / n_vtiles_x) * 32 + lane;
  const long long S = p.S;
  const int state = p.st[s];
  if (w == 0) {
    sred[lane] = 0;       // weight of the tile's variables, per slot
    sred[32 + lane] = 0;  // non-integral flag, per slot
  }
  __syncthreads();
  if (i < p.n_vars && state != kSlotEmpty) {
    const long long f = p.frame[s];
    if (state == kSlotRetiring) {
      // Output statistics of the final iterate x_t (make_output, :92-105).
      const T xv = p.x[i * S + s];
      const bool h = xv > T(0.5);
      if (p.x_out) p.x_out[f * p.ld_x + i] = xv;
      if (p.hard_out) p.hard_out[f * p.ld_hard + i] = h;
      if (h) atomicAdd_block(sred + lane, 1);
      if (!(vmin(fabs(xv), fabs(T(1) - xv)) <= T(1e-5))) atomicOr_block(sred + 32 + lane, 1);
    } else {
      T g;
      T acc = T(0);
      int deg = 0;
      if (state == kSlotFresh) {
        const T gi = p.synth.kind != 0 ? static_cast<T>(synth_llr(p.synth, p.synth.trial0 + f, i))
                                        : p.gamma[f * p.ld_gamma + i];
        g = div_rn(gi, p.mu);
        p.gm[i * S + s] = g;
      } else {
        g = p.gm[i * S + s];
      }
      int ev[DVMAX];
#pragma unroll
      for (int j = 0; j < DVMAX; ++j)  // warp-uniform, increasing edge id, -1 = unused
        ev[j] = j < p.dvmax ? __ldg(p.var_edge + i * p.dvmax + j) : -1;
      T mv[DVMAX];
#pragma unroll
      for (int j = 0; j < DVMAX; ++j) {
        deg += ev[j] >= 0;
        mv[j] = (ev[j] >= 0 && state == kSlotRunning) ? p.msg[(long long)ev[j] * S + s] : T(0);
      }
#pragma unroll
      for (int j = 0; j < DVMAX; ++j)
        if (ev[j] >= 0) acc = add_rn(acc, mv[j]);
      T xv;
      if (deg > 0) {
        xv = clip01(div_rn(sub_rn(acc, g), T(deg)));
      } else {
        xv = g < T(0) ? T(1) : T(0);
      }
      p.x[i * S + s] = xv;
    }
  }
  __syncthreads();
  if (w == 0 && state == kSlotRetiring) {
    if (sred[lane]) atomicAdd(p.weight + s, sred[lane]);
    if (sred[32 + lane]) atomicOr(p.nonint + s, 1);
  }
}

template <typename T, int D, bool REG>
__device__ __forceinline__ void stream_phase_c(const StreamParams<T>& p, int tile, int n_ctiles_x, T* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int cblk = tile % n_ctiles_x;
  const int c = cblk * kStreamCK + w;
  const int s = (tile / n_ctiles_x) * 32 + lane;
  const long long S = p.S;
  const int state = p.st[s];
  T primal = T(0), moved = T(0);
  if (c < p.n_checks && (state == kSlotFresh || state == kSlotRunning)) {
    int vidx[D];
    int d = 0;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      vidx[k] = __ldg(p.chk_var + k * p.m_pad + c);
      d += vidx[k] >= 0;
    }
    const long long e0 = __ldg(p.edge_base + c);
    T gx[D], w_[D], u[D], zn[D], z[D], lam[D];
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const bool on = k < d;
      gx[k] = on ? p.x[(long long)vidx[k] * S + s] : T(0);
      z[k] = T(0);
      lam[k] = T(0);
      if (on && state == kSlotRunning) {
        const long long e = e0 + k;
        if constexpr (sizeof(T) == 4) {
          const float2 v = reinterpret_cast<const float2*>(p.zl)[e * S + s];
          z[k] = v.x;
          lam[k] = v.y;
        } else {
          const double2 v = reinterpret_cast<const double2*>(p.zl)[e * S + s];
          z[k] = v.x;
          lam[k] = v.y;
        }
      }
      w_[k] = add_rn(mul_rn(p.rho, gx[k]), mul_rn(p.one_minus_rho, z[k]));
      u[k] = on ? add_rn(w_[k], lam[k]) : -Num<T>::inf();  // lam holds the scaled dual lambda/mu
    }
    if constexpr (REG) {
      project_pp_fixed<T, D>(u, zn);
    } else {
      project_pp<T, D>(u, zn, d);
    }
#pragma unroll
    for (int k = 0; k < D; ++k) {
      if (k < d) {
        const T r1 = sub_rn(gx[k], zn[k]);
        const T r2 = sub_rn(zn[k], z[k]);
        primal = add_rn(primal, mul_rn(r1, r1));
        moved = add_rn(moved, mul_rn(r2, r2));
        const T lnew = add_rn(lam[k], sub_rn(w_[k], zn[k]));
        const long long e = e0 + k;
        if constexpr (sizeof(T) == 4) {
          reinterpret_cast<float2*>(p.zl)[e * S + s] = make_float2(zn[k], lnew);
        } else {
          reinterpret_cast<double2*>(p.zl)[e * S + s] = make_double2(zn[k], lnew);
        }
        p.msg[e * S + s] = sub_rn(zn[k], lnew);
      }
    }
  } else if (c < p.n_checks && state == kSlotRetiring) {
    // Syndrome of the final hard decision (is_codeword, codes.py:145-154).
    int par = 0;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const int v = __ldg(p.chk_var + k * p.m_pad + c);
      if (v >= 0) par ^= p.x[(long long)v * S + s] > T(0.5);
    }
    primal = par ? T(1) : T(0);  // OR-reduced over the tile through the partial-sum path below
  }
  // Per-slot partial over the tile's checks, fixed order -> deterministic.
  red[w * 32 + lane] = primal;
  red[(kStreamCK + w) * 32 + lane] = moved;
  __syncthreads();
  if (w == 0) {
    T a = red[lane], b = red[kStreamCK * 32 + lane];
#pragma unroll
    for (int q = 1; q < kStreamCK; ++q) {
      a = add_rn(a, red[q * 32 + lane]);
      b = add_rn(b, red[(kStreamCK + q) * 32 + lane]);
    }
    if (state == kSlotRetiring && a > T(0)) atomicOr(p.odd + s, 1);
    if (state == kSlotFresh || state == kSlotRunning) {
      p.part[((long long)cblk * S + s) * 2] = a;
      p.part[((long long)cblk * S + s) * 2 + 1] = b;
      if (a >= p.thr || b >= p.thr) atomicOr(p.notconv + s, 1);
    }
  }
  __syncthreads();
}

// Pop the next frame into slot s (or empty it).
template <typename T>
__device__ __forceinline__ void stream_refill(const StreamParams<T>& p, int s) {
  const int f = atomicAdd(p.ctr + 0, 1);
  p.tcount[s] = 0;
  p.notconv[s] = 0;
  p.weight[s] = 0;
  p.nonint[s] = 0;
  p.odd[s] = 0;
  p.conv[s] = 0;
  if (f < p.batch) {
    p.frame[s] = f;
    p.st[s] = kSlotFresh;
  } else {
    p.frame[s] = -1;
    p.st[s] = kSlotEmpty;
    atomicSub(p.ctr + 1, 1);
  }
}

template <typename T>
__device__ __forceinline__ void stream_phase_s(const StreamParams<T>& p, int s, int n_cblk) {
  // One warp per slot.  Slot fields are read by lane 0 and broadcast, so a
  // lane that runs late can never observe lane 0's updates (the warp's
  // control flow stays uniform around the shuffles below).
  const int lane = threadIdx.x & 31;
  const int state = __shfl_sync(0xffffffffu, lane == 0 ? p.st[s] : 0, 0);
  const int nc = __shfl_sync(0xffffffffu, lane == 0 ? p.notconv[s] : 0, 0);
  __syncwarp();
  if (state == kSlotEmpty) return;
  if (state == kSlotRetiring) {
    if (lane == 0) {
      const long long f = p.frame[s];
      if (p.iters_out) p.iters_out[f] = p.tcount[s];
      if (p.flags_out)
        p.flags_out[f] = (p.conv[s] ? 1 : 0) | (p.nonint[s] ? 0 : 2) | (p.odd[s] ? 0 : 4);
      if (p.weight_out) p.weight_out[f] = p.weight[s];
      stream_refill(p, s);
    }
    return;
  }
  // FRESH or RUNNING: one iteration just completed.
  bool converged = false;
  if (nc == 0) {
    // Exact residual sums (admm_decoder.py:174-176), fixed reduction tree.
    const long long S = p.S;
    double a = 0.0, b = 0.0;  // per-block partials accumulated in fp64
    for (int q = lane; q < n_cblk; q += 32) {
      a += static_cast<double>(p.part[((long long)q * S + s) * 2]);
      b += static_cast<double>(p.part[((long long)q * S + s) * 2 + 1]);
    }
    a = warp_allsum(a);
    b = warp_allsum(b);
    converged = a < p.thr_d && b < p.thr_d;
  }
  if (lane == 0) {
    const int t = p.tcount[s] + 1;
    p.tcount[s] = t;
    p.notconv[s] = 0;
    if (converged || t >= p.t_max) {
      p.conv[s] = converged;
      p.st[s] = kSlotRetiring;
    } else {
      p.st[s] = kSlotRunning;
    }
  }
}

template <typename T, int D, int DVMAX, bool REG>
__global__ void __launch_bounds__(kStreamThreads, 4) streaming_decode_kernel(const StreamParams<T> p) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ T red[2 * kStreamCK * 32];
  __shared__ int sred[64];
  const int n_sw = p.S / 32;
  const int n_vtx = (p.n_vars + kStreamVK - 1) / kStreamVK;
  const int n_ctx = (p.n_checks + kStreamCK - 1) / kStreamCK;
  const int n_vt = n_vtx * n_sw, n_ct = n_ctx * n_sw;
  const int gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int n_gwarp = (gridDim.x * blockDim.x) >> 5;

  // Prologue: every slot takes a frame.
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    p.ctr[0] = 0;
    p.ctr[1] = p.S;
    p.ctr[2] = 0;
  }
  grid.sync();
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < p.S; s += gridDim.x * blockDim.x) stream_refill(p, s);
  grid.sync();

  const long long max_passes = ((long long)(p.batch + p.S - 1) / p.S + 1) * ((long long)p.t_max + 2) + 4;
  for (long long pass = 0; pass < max_passes; ++pass) {
    if (*(volatile int*)(p.ctr + 1) == 0) break;
    for (int tile = blockIdx.x; tile < n_vt; tile += gridDim.x) stream_phase_v<T, D, DVMAX>(p, tile, n_vtx, sred);
    grid.sync();
    for (int tile = blockIdx.x; tile < n_ct; tile += gridDim.x) stream_phase_c<T, D, REG>(p, tile, n_ctx, red);
    grid.sync();
    for (int s = gwarp; s < p.S; s += n_gwarp) stream_phase_s(p, s, n_ctx);
    grid.sync();
  }
}

}  // namespace admm
