// Flooding sum-product BP on the resident engine -- SURVEY.md 8f #4, the
// comparison baseline of the paper's experiments.
//
// Contract: the reference's posterior_llrs / decode_bp (bp_decoder.py:55-112)
// with its check-node rule _check_node_update (:37-52):
//   totals  = gamma + sum_{e in v} c2v_e            (bincount, edge order)
//   v2c_e   = clip(totals[v_e] - c2v_e, +-clip)
//   t_e     = tanh(clip(v2c_e / 2, +-clip / 2))
//   c2v_e   = clip(2 atanh(clip(left_e * right_e, +-(1 - 1e-15))), +-clip)
//             left / right = prefix / suffix products in the row (cumprod order)
//   beliefs = gamma + sum_{e in v} c2v_e
//   early stop after iteration t when every belief is non-zero and the hard
//   decision (belief < 0) satisfies every check.
//
// Mapping: one CTA per frame (persistent, atomic frame queue) exactly like
// resident_decode_kernel; a thread owns CPT checks whose c2v messages stay in
// registers and are mirrored to a slot-major shared buffer for the variable
// pass.  One variable pass computes the totals of iteration t+1 -- which are
// also the beliefs after iteration t -- so the early-stop test rides on the
// next check pass and its barrier (the parity of the beliefs is formed by the
// check threads while they gather the totals anyway).
#pragma once

#include "resident.cuh"

namespace admm {

template <typename T>
struct BpParams {
  int n_vars, n_checks, m_pad;
  const int* chk_var;       // [D][m_pad] original variable of slot k of check c, -1 = unused
  const uint16_t* var_pos;  // [n_vars][DVMAX] positions k * m_pad + c of the variable's edges
  const uint8_t* var_deg;
  long long batch;
  const T* gamma;
  long long ld_gamma;
  T clip, half_clip, guard;
  int t_max, early_stop;
  T* beliefs_out;
  long long ld_beliefs;
  T* x_out;  // bit-1 probabilities
  long long ld_x;
  uint8_t* hard_out;
  long long ld_hard;
  int* iters_out;
  uint8_t* flags_out;
  int* weight_out;
  int* queue;
  SynthParams synth;
};

__device__ __forceinline__ float bp_tanh(float v) { return tanhf(v); }
__device__ __forceinline__ double bp_tanh(double v) { return tanh(v); }
__device__ __forceinline__ float bp_atanh(float v) { return atanhf(v); }
__device__ __forceinline__ double bp_atanh(double v) { return atanh(v); }
template <typename T> __device__ __forceinline__ T clip_pm(T v, T c) { return vmin(vmax(v, -c), c); }

// Shared memory: msg[D][m_pad] | totals[N] | gamma[N] | pos[N][DVMAX] | deg[N] | red
struct BpSmem {
  int msg, tot, gam, pos, deg, red, total;
  __host__ __device__ static int align16(int b) { return (b + 15) & ~15; }
  __host__ __device__ BpSmem(int elem, int n_vars, int msg_len, int dvmax) {
    msg = 0;
    tot = align16(msg + elem * msg_len);
    gam = align16(tot + elem * n_vars);
    pos = align16(gam + elem * n_vars);
    deg = align16(pos + 2 * dvmax * n_vars);
    red = align16(deg + n_vars);
    total = align16(red + 16);
  }
};

template <typename T, int D, int CPT, int DVMAX>
__global__ void __launch_bounds__(512) bp_decode_kernel(const BpParams<T> p) {
  using Pos = typename VarPos<DVMAX>::type;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int N = p.n_vars, M = p.n_checks, MP = p.m_pad;
  const BpSmem L(sizeof(T), N, D * MP, DVMAX);
  T* msg = reinterpret_cast<T*>(smem_raw + L.msg);
  T* tot = reinterpret_cast<T*>(smem_raw + L.tot);
  T* gam = reinterpret_cast<T*>(smem_raw + L.gam);
  Pos* spos = reinterpret_cast<Pos*>(smem_raw + L.pos);
  uint8_t* sdeg = reinterpret_cast<uint8_t*>(smem_raw + L.deg);
  int* s_frame = reinterpret_cast<int*>(smem_raw + L.red);
  int* s_weight = s_frame + 1;
  const int tid = threadIdx.x, NT = blockDim.x, lane = tid & 31;

  for (int i = tid; i < N; i += NT) {
    spos[i] = reinterpret_cast<const Pos*>(p.var_pos)[i];
    sdeg[i] = p.var_deg[i];
  }
  int vidx[CPT][D];
#pragma unroll
  for (int q = 0; q < CPT; ++q) {
    const int c = tid + q * NT;
#pragma unroll
    for (int k = 0; k < D; ++k) vidx[q][k] = (c < M) ? __ldg(p.chk_var + k * MP + c) : -1;
  }
  T c2v[CPT][D];

  for (;;) {
    __syncthreads();
    if (tid == 0) {
      *s_frame = atomicAdd(p.queue, 1);
      *s_weight = 0;
    }
    __syncthreads();
    const long long f = *s_frame;
    if (f >= p.batch) break;

    for (int i = tid; i < N; i += NT) gam[i] = frame_llr<T>(p, f, i);
#pragma unroll
    for (int q = 0; q < CPT; ++q) {
      const int c = tid + q * NT;
#pragma unroll
      for (int k = 0; k < D; ++k) {
        c2v[q][k] = T(0);
        if (vidx[q][k] >= 0) msg[k * MP + c] = T(0);
      }
    }
    __syncthreads();

    int t = 0;
    bool found = false;
    for (;;) {
      // ---- variable pass: totals = gamma + bincount(c2v) = beliefs after t iterations ----
      bool zero = false;
      for (int i = tid; i < N; i += NT) {
        const Pos ps = spos[i];
        const int dg = sdeg[i];
        T acc = T(0);
#pragma unroll
        for (int j = 0; j < DVMAX; ++j)
          if (j < dg) acc = add_rn(acc, msg[unpack_pos(ps, j)]);
        const T b = add_rn(gam[i], acc);
        tot[i] = b;
        zero |= b == T(0);
      }
      __syncthreads();
      // ---- check pass: parity of the beliefs, then the tanh-rule update ----
      const bool last = t == p.t_max;
      bool odd = false;
#pragma unroll
      for (int q = 0; q < CPT; ++q) {
        const int c = tid + q * NT;
        if (c >= M) continue;
        T tv[D], th[D];
        int par = 0;
#pragma unroll
        for (int k = 0; k < D; ++k) {
          tv[k] = vidx[q][k] >= 0 ? tot[vidx[q][k]] : T(0);
          par ^= vidx[q][k] >= 0 && tv[k] < T(0);
        }
        odd |= par;
        if (last) continue;
#pragma unroll
        for (int k = 0; k < D; ++k) {
          const T v2c = clip_pm(sub_rn(tv[k], c2v[q][k]), p.clip);
          th[k] = vidx[q][k] >= 0 ? bp_tanh(clip_pm(mul_rn(T(0.5), v2c), p.half_clip)) : T(1);
        }
        // leave-one-out products: prefix (left) times suffix (right), each
        // accumulated in the reference's cumprod order
        T left[D], right[D];
        left[0] = T(1);
#pragma unroll
        for (int k = 1; k < D; ++k) left[k] = k == 1 ? th[0] : mul_rn(left[k - 1], th[k - 1]);
        // suffix of the ACTIVE row: the reference's row ends at its degree, so
        // padded slots (th = 1) must not start the product chain
        int deg = 0;
#pragma unroll
        for (int k = 0; k < D; ++k) deg += vidx[q][k] >= 0;
        T run = T(1);
        bool started = false;
#pragma unroll
        for (int k = D - 1; k >= 0; --k) {
          right[k] = run;
          if (k < deg) {
            run = started ? mul_rn(run, th[k]) : th[k];
            started = true;
          }
        }
#pragma unroll
        for (int k = 0; k < D; ++k) {
          if (vidx[q][k] < 0) continue;
          const T prod = clip_pm(k == 0 ? right[0] : (k == deg - 1 ? left[k] : mul_rn(left[k], right[k])), p.guard);
          const T m = clip_pm(mul_rn(T(2), bp_atanh(prod)), p.clip);
          c2v[q][k] = m;
          msg[k * MP + c] = m;
        }
      }
      const int stop_any = __syncthreads_or(odd || zero);
      if (t >= 1 && p.early_stop && !stop_any) {
        found = true;
        break;
      }
      if (last) break;
      ++t;
    }

    // ---- outputs (decode_bp, bp_decoder.py:98-112) ----
    bool integral = true;
    int ones = 0;
    for (int i = tid; i < N; i += NT) {
      const T b = tot[i];
      const T p1 = mul_rn(T(0.5), sub_rn(T(1), bp_tanh(mul_rn(T(0.5), b))));
      const bool h = b < T(0);
      ones += h;
      integral &= vmin(p1, sub_rn(T(1), p1)) <= T(1e-5);
      if (p.beliefs_out) p.beliefs_out[f * p.ld_beliefs + i] = b;
      if (p.x_out) p.x_out[f * p.ld_x + i] = p1;
      if (p.hard_out) p.hard_out[f * p.ld_hard + i] = h;
    }
    bool odd = false;
#pragma unroll
    for (int q = 0; q < CPT; ++q) {
      int par = 0;
#pragma unroll
      for (int k = 0; k < D; ++k)
        if (vidx[q][k] >= 0) par ^= tot[vidx[q][k]] < T(0);
      odd |= par;
    }
    ones = __reduce_add_sync(0xffffffffu, ones);
    if (lane == 0 && ones) atomicAdd(s_weight, ones);
    const int all_integral = __syncthreads_and(integral);
    const int any_odd = __syncthreads_or(odd);
    if (tid == 0) {
      if (p.iters_out) p.iters_out[f] = t;
      if (p.flags_out)
        p.flags_out[f] = (found ? kFlagConverged : 0) | (all_integral ? kFlagIntegral : 0) |
                         (any_odd ? 0 : kFlagCodeword);
      if (p.weight_out) p.weight_out[f] = *s_weight;
    }
  }
}

}  // namespace admm
