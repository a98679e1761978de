// Resident engine: one CTA decodes one frame at a time, entirely on chip.
//
// Mapping of the reference decode loop (admm_decoder.py:152-182):
//   * every thread owns CPT checks; the replicas z and duals lambda of their
//     edges live in REGISTERS for the whole decode (AdmmState, :47-71);
//   * the per-edge messages z - lambda/mu that the x-update averages are
//     written to a shared-memory edge buffer ``msg`` laid out slot-major
//     (msg[k * m_pad + c] = slot k of check c), so a warp's 32 checks store
//     32 consecutive words per slot;
//   * the x-update (:108-124) runs over variables: each thread gathers the
//     messages of its variables' edges (CSC positions packed as 16-bit
//     offsets) in increasing edge order -- the reference's bincount order --
//     and writes x to shared memory;
//   * the z-update (:127-141), the projection (parity_polytope.py:352-421),
//     the residuals (:174-176) and the lambda-update (:144-149) are one fused
//     pass over the thread's checks in registers;
//   * the stop rule (:169,179) is a warp-butterfly + shared-memory reduction
//     whose result is bitwise identical in every thread.
// The CTA is persistent: when its frame converges (or hits t_max) it writes
// the outputs (make_output, :92-105) and pulls the next frame index from a
// global atomic queue, so converged frames retire immediately and the
// heavy-tailed iteration counts never idle an SM.
#pragma once

#include "common.cuh"
#include "projection.cuh"
#include "synth.cuh"

namespace admm {

// Output flag bits per frame.
enum : uint8_t { kFlagConverged = 1, kFlagIntegral = 2, kFlagCodeword = 4 };

template <typename T>
struct ResidentParams {
  // graph (device, immutable)
  int n_vars, n_checks, m_pad;
  const int* chk_var;         // [D][m_pad]  variable of slot k of check c, -1 = unused
  const uint16_t* var_pos;    // [n_vars][DVMAX] msg positions of the variable's edges
  const uint8_t* var_deg;     // [n_vars]
  const int* edge_base;       // [n_checks]  reference edge id of slot 0 (check_ptr)
  const int* var_orig;        // regular kernel: internal variable -> original variable (null = identity)
  const int* edge_ref;        // regular kernel: [check][D] reference edge id of slot k (null = c*D + k)
  const int* check_rot;       // colored regular kernel, D mod DV = 1: rotation of each check (null = 0)
  // frames
  long long batch;
  const T* gamma;
  long long ld_gamma;
  // parameters
  // thr_d = eps^2 E (admm_decoder.py:169) in fp64: the exact stop-rule sums
  // are accumulated and compared in fp64 in both modes.  thr is its T value
  // rounded UP, so a per-thread partial >= thr implies partial >= thr_d.
  T mu, inv_mu, rho, one_minus_rho, thr;
  double thr_d;
  // fp32 regular kernel: the exact stop-rule sums as 42-bit fixed point
  // (fx_sum below): fx_scale = 2^k with thr * fx_scale in [2^20, 2^21),
  // fx_thr = ceil(thr_d * fx_scale * 2^21).
  float fx_scale;
  unsigned long long fx_thr;
  int t_max;
  // optional initial state (reference edge order), null = zeros
  const T* z_in;
  const T* lam_in;
  long long ld_edge;
  // outputs (any may be null)
  T* x_out;
  long long ld_x;
  uint8_t* hard_out;
  long long ld_hard;
  int* iters_out;
  uint8_t* flags_out;
  int* weight_out;
  T* z_out;
  T* lam_out;
  // work queue
  int* queue;
  // fused frame synthesis (kind 0 = read gamma)
  SynthParams synth;
};

// LLR of variable i of frame f: from memory, or synthesised from
// (seed, point, trial0 + f) when the call asked for fused synthesis.
template <typename T, typename P>
__device__ __forceinline__ T frame_llr(const P& p, long long f, int i) {
  if (p.synth.kind != 0) return static_cast<T>(synth_llr(p.synth, p.synth.trial0 + f, i));
  return p.gamma[f * p.ld_gamma + i];
}

template <int DVMAX>
struct VarPos;
template <> struct VarPos<4> { using type = uint2; };
template <> struct VarPos<8> { using type = uint4; };

__device__ __forceinline__ int unpack_pos(const uint2& p, int j) {
  const unsigned w = (j < 2) ? p.x : p.y;
  return (j & 1) ? (w >> 16) : (w & 0xffffu);
}
__device__ __forceinline__ int unpack_pos(const uint4& p, int j) {
  const unsigned w = (j < 2) ? p.x : (j < 4) ? p.y : (j < 6) ? p.z : p.w;
  return (j & 1) ? (w >> 16) : (w & 0xffffu);
}

// Shared-memory carve-up (bytes), computed identically on host and device.
struct ResidentSmem {
  int msg, x, gm, ideg, pos, deg, red, total;
  __host__ __device__ static int align16(int b) { return (b + 15) & ~15; }
  __host__ __device__ ResidentSmem(int elem, int n_vars, int msg_len, int dvmax) {
    msg = 0;
    x = align16(msg + elem * msg_len);
    gm = align16(x + elem * n_vars);
    ideg = align16(gm + elem * n_vars);  // variable degree as T
    pos = align16(ideg + elem * n_vars);
    deg = align16(pos + 2 * dvmax * n_vars);
    red = align16(deg + n_vars);
    total = align16(red + 8 * 2 * 32 + 16);  // fp64 reduction slots
  }
};

template <typename T, int D, int CPT, int DVMAX>
__global__ void __launch_bounds__(512) resident_decode_kernel(const ResidentParams<T> p) {
  using Pos = typename VarPos<DVMAX>::type;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int N = p.n_vars, M = p.n_checks, MP = p.m_pad;
  const ResidentSmem L(sizeof(T), N, D * MP, DVMAX);
  T* msg = reinterpret_cast<T*>(smem_raw + L.msg);
  T* xs = reinterpret_cast<T*>(smem_raw + L.x);
  T* gm = reinterpret_cast<T*>(smem_raw + L.gm);
  T* ideg = reinterpret_cast<T*>(smem_raw + L.ideg);
  Pos* spos = reinterpret_cast<Pos*>(smem_raw + L.pos);
  uint8_t* sdeg = reinterpret_cast<uint8_t*>(smem_raw + L.deg);
  double* red = reinterpret_cast<double*>(smem_raw + L.red);
  int* s_frame = reinterpret_cast<int*>(smem_raw + L.red + sizeof(double) * 64);
  int* s_weight = s_frame + 1;

  const int tid = threadIdx.x, NT = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nwarps = NT >> 5;

  // ---- graph staging (once per CTA) ----
  for (int i = tid; i < N; i += NT) {
    spos[i] = reinterpret_cast<const Pos*>(p.var_pos)[i];
    const int dg = p.var_deg[i];
    sdeg[i] = static_cast<uint8_t>(dg);
    ideg[i] = T(dg > 0 ? dg : 1);
  }
  int vidx[CPT][D];
  int cdeg[CPT];
#pragma unroll
  for (int q = 0; q < CPT; ++q) {
    const int c = tid + q * NT;
    cdeg[q] = 0;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      vidx[q][k] = (c < M) ? __ldg(p.chk_var + k * MP + c) : -1;
      cdeg[q] += vidx[q][k] >= 0;
    }
  }

  T z[CPT][D], lam[CPT][D];

  for (;;) {
    __syncthreads();  // previous frame fully consumed (smem reuse, s_frame)
    if (tid == 0) {
      *s_frame = atomicAdd(p.queue, 1);
      *s_weight = 0;
    }
    __syncthreads();
    const long long f = *s_frame;
    if (f >= p.batch) break;

    // ---- frame setup: gamma/mu, zero (or given) state, messages ----
    for (int i = tid; i < N; i += NT) gm[i] = div_rn(frame_llr<T>(p, f, i), p.mu);
#pragma unroll
    for (int q = 0; q < CPT; ++q) {
      const int c = tid + q * NT;
#pragma unroll
      for (int k = 0; k < D; ++k) {
        T z0 = T(0), l0 = T(0);
        if (p.z_in != nullptr && vidx[q][k] >= 0) {
          const long long e = f * p.ld_edge + p.edge_base[c] + k;
          z0 = p.z_in[e];
          l0 = div_rn(p.lam_in[e], p.mu);  // duals kept scaled: lambda / mu
        }
        z[q][k] = z0;
        lam[q][k] = l0;
        if (vidx[q][k] >= 0) msg[k * MP + c] = sub_rn(z0, l0);
      }
    }
    __syncthreads();

    int t = 0;
    bool converged = false;
    while (t < p.t_max) {
      ++t;
      // ---- x-update (admm_decoder.py:108-124) ----
      for (int i = tid; i < N; i += NT) {
        const Pos ps = spos[i];
        const int dg = sdeg[i];
        T acc = T(0);
#pragma unroll
        for (int j = 0; j < DVMAX; ++j)
          if (j < dg) acc = add_rn(acc, msg[unpack_pos(ps, j)]);
        T xv;
        if (dg > 0) {
          xv = clip01(div_rn(sub_rn(acc, gm[i]), ideg[i]));
        } else {
          xv = gm[i] < T(0) ? T(1) : T(0);
        }
        xs[i] = xv;
      }
      __syncthreads();

      // ---- fused z-update + projection + residuals + lambda-update ----
      T primal = T(0), moved = T(0);
#pragma unroll
      for (int q = 0; q < CPT; ++q) {
        const int c = tid + q * NT;
        if (c < M) {
          T gx[D], w[D], u[D], zn[D];
#pragma unroll
          for (int k = 0; k < D; ++k) {
            const bool on = vidx[q][k] >= 0;
            gx[k] = on ? xs[vidx[q][k]] : T(0);
            w[k] = add_rn(mul_rn(p.rho, gx[k]), mul_rn(p.one_minus_rho, z[q][k]));
            u[k] = on ? add_rn(w[k], lam[q][k]) : -Num<T>::inf();
          }
          project_pp<T, D>(u, zn, cdeg[q]);
#pragma unroll
          for (int k = 0; k < D; ++k) {
            if (vidx[q][k] >= 0) {
              const T r1 = sub_rn(gx[k], zn[k]);
              const T r2 = sub_rn(zn[k], z[q][k]);
              primal = add_rn(primal, mul_rn(r1, r1));
              moved = add_rn(moved, mul_rn(r2, r2));
              lam[q][k] = add_rn(lam[q][k], sub_rn(w[k], zn[k]));
              z[q][k] = zn[k];
              msg[k * MP + c] = sub_rn(zn[k], lam[q][k]);
            }
          }
        }
      }
      // ---- stop rule (admm_decoder.py:169,174-181): fp64 accumulation ----
      const double pa = warp_allsum(static_cast<double>(primal));
      const double pb = warp_allsum(static_cast<double>(moved));
      if (lane == 0) {
        red[2 * warp] = pa;
        red[2 * warp + 1] = pb;
      }
      __syncthreads();
      double a = lane < nwarps ? red[2 * lane] : 0.0;
      double b = lane < nwarps ? red[2 * lane + 1] : 0.0;
      a = warp_allsum(a);
      b = warp_allsum(b);
      if (a < p.thr_d && b < p.thr_d) {
        converged = true;
        break;
      }
    }

    // ---- outputs (make_output, admm_decoder.py:92-105; is_codeword, codes.py:145-154) ----
    bool integral = true;
    int ones = 0;
    for (int i = tid; i < N; i += NT) {
      const T xv = xs[i];
      const bool h = xv > T(0.5);
      ones += h;
      integral &= vmin(fabs(xv), fabs(T(1) - xv)) <= T(1e-5);
      if (p.x_out) p.x_out[f * p.ld_x + i] = xv;
      if (p.hard_out) p.hard_out[f * p.ld_hard + i] = h;
    }
    bool odd = false;
#pragma unroll
    for (int q = 0; q < CPT; ++q) {
      const int c = tid + q * NT;
      int par = 0;
#pragma unroll
      for (int k = 0; k < D; ++k)
        if (vidx[q][k] >= 0) par ^= (xs[vidx[q][k]] > T(0.5));
      odd |= (c < M) && par;
      if (p.z_out && c < M) {
#pragma unroll
        for (int k = 0; k < D; ++k) {
          if (vidx[q][k] >= 0) {
            const long long e = f * p.ld_edge + p.edge_base[c] + k;
            p.z_out[e] = z[q][k];
            p.lam_out[e] = mul_rn(p.mu, lam[q][k]);
          }
        }
      }
    }
    ones = __reduce_add_sync(0xffffffffu, ones);
    if (lane == 0 && ones) atomicAdd(s_weight, ones);
    const int all_integral = __syncthreads_and(integral);
    const int any_odd = __syncthreads_or(odd);
    if (tid == 0) {
      if (p.iters_out) p.iters_out[f] = t;
      if (p.flags_out)
        p.flags_out[f] = (converged ? kFlagConverged : 0) | (all_integral ? kFlagIntegral : 0) |
                         (any_odd ? 0 : kFlagCodeword);
      if (p.weight_out) p.weight_out[f] = *s_weight;
    }
  }
}

}  // namespace admm
