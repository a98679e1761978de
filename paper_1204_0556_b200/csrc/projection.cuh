// Exact Euclidean projection onto the parity polytope PP_d, in registers.
//
// Contract: the reference's project_batch (parity_polytope.py:352-421).
//   v  = u sorted descending (stable)                      :366-367
//   c  = clip(v, 0, 1); r = 2 floor(sum c / 2), r <= d       :368-372
//   f  = +1 on the top r+1 coordinates, -1 elsewhere          :374
//   fz = 2 * sum_{k<=r} c_k - sum c                           :375-376
//   beta_max = (v_r - v_{r+1}) / 2, or v_r when r = d-1       :378-380
//   inside (return c) when r >= d, fz <= r + TOL, beta_max<=0 :382
//   otherwise z = clip(v - beta f, 0, 1) with beta the root of
//   g(beta) = f . clip(v - beta f, 0, 1) = r on [0, beta_max], capped at
//   beta_max when g stays above r                             :385-414
//
// B200 formulation (no grid, no permutation).  Writing s_k for the shift at
// which coordinate k enters the open band (0,1) -- s_k = u_k - 1 on the +1
// block and s_k = -u_k on the -1 block -- every coordinate is active on
// exactly (s_k, s_k + 1), so g(beta) = (r + 1) - sum_k clip(beta - s_k, 0, 1)
// and g(beta) = r  <=>  sum_k max(beta - s_k, 0) = 1 below the root.  That is
// water-filling: with s sorted ascending and P_j = 1 + s_(1) + ... + s_(j),
// every partial line (P_j)/j over-estimates the root and the active prefix
// attains it, so
//          beta* = min(beta_max, min_j P_j / j).
// Two value-only sorting networks (no index payload: f is recovered as
// u_k >= v_r, exact whenever the row is projected because v_r > v_{r+1}
// then) and one prefix scan replace the reference's O(d^2) grid evaluation.
// The result agrees with project_batch to rounding (tests/test_projection*).
//
// Degree handling: arrays are sized D (a compile-time bucket); the active
// degree d <= D is a runtime value and padded slots must hold -inf in u.
#pragma once

#include "common.cuh"
#include "sortnet.cuh"

namespace admm {

// Sum of c[0..d) in numpy's pairwise_sum order for short rows: sequential
// below 8 elements, eight interleaved partial sums combined as a tree and a
// sequential tail otherwise.  Zeros in padded slots leave the sequential sum
// unchanged.  Only matters at rounding level (it fixes r = even floor of the
// l1 norm bit-exactly in fp64 where the norm sits on an even integer).
template <typename T, int D>
__device__ __forceinline__ T numpy_rowsum(const T (&c)[D], int d) {
  T seq = c[0];
#pragma unroll
  for (int k = 1; k < D; ++k) seq = add_rn(seq, c[k]);
  if constexpr (D < 8) {
    return seq;
  } else {
    T acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = c[j];
    // Full blocks of eight beyond the first (numpy adds block i into lane j).
    constexpr int kBlocks = D / 8;
#pragma unroll
    for (int b = 1; b < kBlocks; ++b) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const bool in = (b * 8 + 8) <= d;  // block fully inside the active row
        if (in) acc[j] = add_rn(acc[j], c[b * 8 + j]);
      }
    }
    T res = add_rn(add_rn(add_rn(acc[0], acc[1]), add_rn(acc[2], acc[3])),
                   add_rn(add_rn(acc[4], acc[5]), add_rn(acc[6], acc[7])));
    const int tail0 = (d / 8) * 8;
#pragma unroll
    for (int k = 8; k < D; ++k)
      if (k >= tail0) res = add_rn(res, c[k]);
    return d < 8 ? seq : res;
  }
}

// ---------------------------------------------------------------------------
// Cut-search formulation (round 2): one sorting network, no order statistics.
//
// With d_k = u_k - 1/2 the candidate facet is T = {k : d_k >= 0}, made odd by
// moving the coordinate closest to 1/2 across when |T| is even; whenever the
// cube clip lies outside PP_d this T is the reference's f_r (:374 -- a
// violated facet is unique, and all but at most the moved coordinate sit on
// their own side of 1/2).  The activation shift of coordinate k,
// s_k = u_k - 1 on T and -u_k off T, is then |d_k| - 1/2, except for the moved
// coordinate where it is -|d_k| - 1/2 -- the smallest of all.  So ONE
// ascending sort of |d_k| yields the water-filling prefixes
// P_j = 1 + s_(1) + ... + s_(j) directly, and
//          beta* = max(0, min_j P_j / j):
// min_j P_j / j <= 0 exactly when sum_k max(-s_k, 0) >= 1, i.e. when the
// facet is NOT violated (the facet test :375-382; then beta = 0 and the
// result is the cube clip), and beta* <= beta_max always holds for the exact
// root (the reference's cap :378-380 only guards its grid search).  The sign
// of each coordinate's shift is sign(d_k), inverted for the moved coordinate,
// which is recognised by |d_k| == min |d| (a tie moves both: then the
// distances of the two to their vertices already sum to 1 and beta* = 0).
// Versus the two-network version above: no second network (7 / 22
// compare-exchanges at D = 6 / 13), no r, no order statistics selected by r,
// no facet test: ~85 instead of ~120 instructions per degree-6 check, and half
// the ALU-pipe (FMNMX / select) load the fp32 kernels are bound by.
// Padded slots (u = -inf) have s = +inf, sort last and project to 0.
//
// fp32 (throughput mode): the same computation arranged for the issue-bound
// kernels -- packed FADD2 / FMUL2 for d_k and the shift signs, the prefix
// means as one FFMA each, beta_j = A_j / j + (1 - j / 2) / j with A_j the
// running sum of the sorted |d|, and the sign of each coordinate's shift from
// w_k = d_k (te - |d_k|), te = min |d| (or -1 when nothing moves): te - |d_k|
// is +0 for the moved coordinate and negative otherwise, so w_k carries the
// INVERTED sign of the shift -- FMA-pipe work and one LOP3 per coordinate, no
// compare / select.  (The difference must stay an FADD: ptxas contracts
// mul.rn.f32x2 + sub.rn.f32x2 into FFMA2, so a test on squares, te^2 - d_k^2,
// would not be exactly 0 for the moved coordinate.)
template <int D>
__device__ __forceinline__ void project_pp_cut_f32(const float (&u)[D], float (&z)[D]) {
  float dk[D], t[D];
  uint32_t sx = 0;
  const float2 mhalf = make_float2(-0.5f, -0.5f);
#pragma unroll
  for (int j = 0; j < D / 2; ++j) {
    const float2 d2 = __fadd2_rn(make_float2(u[2 * j], u[2 * j + 1]), mhalf);
    dk[2 * j] = d2.x;
    dk[2 * j + 1] = d2.y;
  }
  if constexpr (D & 1) dk[D - 1] = u[D - 1] - 0.5f;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    sx ^= __float_as_uint(dk[k]);
    t[k] = fabsf(dk[k]);
  }
  SortNet<D>::asc(t);
  const bool even = ((sx >> 31) & 1u) == static_cast<uint32_t>(D & 1);
  float a = even ? -t[0] : t[0];
  float beta = a + 0.5f;
#pragma unroll
  for (int j = 1; j < D; ++j) {
    a += t[j];
    beta = fminf(beta, __fmaf_rn(a, 1.f / (j + 1), (1.f - 0.5f * (j + 1)) / (j + 1)));
  }
  beta = fmaxf(beta, 0.f);
  const float te = even ? t[0] : -1.f;  // |d| >= 0: nothing equals -1
  auto shift = [&](float uk, float w) {
    const float sb = __uint_as_float(__float_as_uint(beta) | (~__float_as_uint(w) & 0x80000000u));
    return __saturatef(uk - sb);
  };
#pragma unroll
  for (int j = 0; j < D / 2; ++j) {
    const float2 d2 = make_float2(dk[2 * j], dk[2 * j + 1]);
    const float2 w2 = __fmul2_rn(d2, make_float2(te - fabsf(d2.x), te - fabsf(d2.y)));
    z[2 * j] = shift(u[2 * j], w2.x);
    z[2 * j + 1] = shift(u[2 * j + 1], w2.y);
  }
  if constexpr (D & 1) z[D - 1] = shift(u[D - 1], dk[D - 1] * (te - fabsf(dk[D - 1])));
}

template <typename T, int D>
__device__ __forceinline__ void project_pp_cut(const T (&u)[D], T (&z)[D]) {
  if constexpr (sizeof(T) == 4) {
    project_pp_cut_f32<D>(u, z);
    return;
  } else {
  T dk[D], t[D];
  uint32_t sx = 0;  // bit 31: parity of the coordinates below 1/2
#pragma unroll
  for (int k = 0; k < D; ++k) {
    dk[k] = sub_rn(u[k], T(0.5));
    sx ^= static_cast<uint32_t>(__double2hiint(dk[k]));
    t[k] = fabs(dk[k]);
  }
  SortNet<D>::asc(t);
  // |T| = D - (coordinates below 1/2) is even: move the closest coordinate
  const bool even = ((sx >> 31) & 1u) == static_cast<uint32_t>(D & 1);
  T p = add_rn(T(0.5), even ? -t[0] : t[0]);  // P_1 = 1 + s_(1)
  T beta = p;
#pragma unroll
  for (int j = 1; j < D; ++j) {
    p = add_rn(p, sub_rn(t[j], T(0.5)));
    beta = vmin(beta, mul_rn(p, T(1) / T(j + 1)));
  }
  beta = vmax(beta, T(0));
  const T te = even ? t[0] : T(-1);  // |d| >= 0: nothing equals -1
#pragma unroll
  for (int k = 0; k < D; ++k) {
    const bool up = (dk[k] >= T(0)) != (fabs(dk[k]) == te);
    z[k] = clip01(up ? sub_rn(u[k], beta) : add_rn(u[k], beta));
  }
  }
}

// Project u (degree d <= D; u[k] = -inf for k >= d) onto PP_d.  z[k] for
// k >= d is left as 0.  Returns true when the facet test sent the row through
// the water-filling search (diagnostics only).
template <typename T, int D>
__device__ __forceinline__ bool project_pp(const T (&u)[D], T (&z)[D], int d) {
#ifndef ADMM_PROJ_TWO_SORT
  project_pp_cut<T, D>(u, z);
  return true;
#endif
  T v[D];
#pragma unroll
  for (int k = 0; k < D; ++k) v[k] = u[k];
  SortNet<D>::desc(v);

  T c[D];
#pragma unroll
  for (int k = 0; k < D; ++k) c[k] = clip01(v[k]);
  const T total = numpy_rowsum<T, D>(c, d);
  int r = 2 * static_cast<int>(floor(total * T(0.5)));
  r = r < d ? r : d;
  const int top = r < d - 1 ? r : d - 1;
  const int nxt = (r + 1) < (d - 1) ? (r + 1) : (d - 1);

  // Order statistics v_top, v_nxt and the head sum sum_{k<=top} c_k, read
  // out of the sorted registers with compile-time indices.
  T v_top = v[0], v_nxt = v[0], head = c[0], run = c[0];
#pragma unroll
  for (int k = 1; k < D; ++k) {
    run = add_rn(run, c[k]);
    if (k == top) { v_top = v[k]; head = run; }
    if (k == nxt) v_nxt = v[k];
  }
  const T fz = sub_rn(mul_rn(T(2), head), total);
  const T beta_max = (r <= d - 2) ? mul_rn(T(0.5), sub_rn(v_top, v_nxt)) : v_top;
  const bool inside = (r >= d) || (fz <= T(r) + Num<T>::kTol) || (beta_max <= T(0));

  if (inside) {
#pragma unroll
    for (int k = 0; k < D; ++k) z[k] = (k < d) ? clip01(u[k]) : T(0);
    return false;
  }

  // Water-filling for the shift beta (see header comment).
  T s[D];
#pragma unroll
  for (int k = 0; k < D; ++k) s[k] = (u[k] >= v_top) ? sub_rn(u[k], T(1)) : -u[k];  // pads: +inf
  SortNet<D>::asc(s);
  T beta = beta_max;
  T p = T(1);
#pragma unroll
  for (int j = 0; j < D; ++j) {
    p = add_rn(p, s[j]);
    beta = vmin(beta, mul_rn(p, T(1) / T(j + 1)));
  }
#pragma unroll
  for (int k = 0; k < D; ++k) {
    const T t = (u[k] >= v_top) ? sub_rn(u[k], beta) : add_rn(u[k], beta);
    z[k] = (k < d) ? clip01(t) : T(0);
  }
  return true;
}

// Bitonic merger (ascending) for a V-shaped sequence of length D, padded
// conceptually to the next power of two with +inf: compare-exchanges that
// touch a padded slot are no-ops and are pruned at compile time (7 for
// D = 6, 22 for D = 13, versus 12 / 48 for a full sorting network).
constexpr int next_pow2(int d) { return d <= 1 ? 1 : 2 * next_pow2((d + 1) / 2); }

template <typename T, int D>
__device__ __forceinline__ void bitonic_merge_asc(T (&s)[D]) {
  constexpr int P = next_pow2(D);
#pragma unroll
  for (int h = P / 2; h >= 1; h /= 2) {
#pragma unroll
    for (int i = 0; i < P; ++i)
      if ((i & h) == 0 && i + h < D) ce_asc(s[i], s[i + h]);
  }
}

#ifndef ADMM_PROJ_FMA_MASK
#define ADMM_PROJ_FMA_MASK 0
#endif

// Fixed-degree variant used by the regular-code kernels: d == D at compile
// time, no padding, and branch-free -- a row that passes the facet test gets
// beta = 0, and clip(u - 0 * f) is exactly the cube clip the reference
// returns for it (:418).  Same contract as project_pp.
template <typename T, int D>
__device__ __forceinline__ void project_pp_fixed(const T (&u)[D], T (&z)[D]) {
#ifndef ADMM_PROJ_TWO_SORT
  project_pp_cut<T, D>(u, z);
  return;
#endif
  T v[D];
#pragma unroll
  for (int k = 0; k < D; ++k) v[k] = u[k];
  SortNet<D>::desc(v);
  T c[D];
#pragma unroll
  for (int k = 0; k < D; ++k) c[k] = clip01(v[k]);
  const T total = numpy_rowsum<T, D>(c, D);
  const int r = 2 * static_cast<int>(floor(total * T(0.5)));
  // Projected rows have r even and r <= D - 1, so r indexes an even slot.
  T v_top = v[0], v_nxt = v[D > 1 ? 1 : 0], head = c[0], run = c[0];
#pragma unroll
  for (int k = 1; k < D; ++k) {
    run = add_rn(run, c[k]);
    if ((k & 1) == 0 && k == r) {
      v_top = v[k];
      v_nxt = v[k + 1 < D ? k + 1 : k];
      head = run;
    }
  }
  const T fz = sub_rn(mul_rn(T(2), head), total);
  const T beta_max = (r <= D - 2) ? mul_rn(T(0.5), sub_rn(v_top, v_nxt)) : v_top;
  const bool inside = (r >= D) || (fz <= T(r) + Num<T>::kTol) || (beta_max <= T(0));

  // Activation shifts in SORTED order: s = v_k - 1 on the +1 block (k <= r,
  // descending) then -v_k (ascending) -- a V-shaped sequence whatever r is,
  // so a bitonic merger sorts it.
  T s[D];
  if constexpr (sizeof(T) == 4 && ADMM_PROJ_FMA_MASK) {
    // fp32 (throughput mode): the block mask as a float on the FMA pipe,
    // m_k = [k <= r] = sat(r + 1 - k), and s_k = m_k (2 v_k - 1) - v_k, in
    // place of integer compares and selects on the ALU pipe (the kernel is
    // ALU-issue bound).  Same values up to the rounding of 2 v_k - 1.
    const float rp1 = static_cast<float>(r + 1);
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const float m = __saturatef(rp1 - static_cast<float>(k));
      s[k] = __fmaf_rn(m, __fmaf_rn(2.f, v[k], -1.f), -v[k]);
    }
  } else {
    const int r2 = r >> 1;
#pragma unroll
    for (int k = 0; k < D; ++k) s[k] = (((k + 1) >> 1) <= r2) ? sub_rn(v[k], T(1)) : -v[k];
  }
  bitonic_merge_asc<T, D>(s);
  T beta = beta_max, p = T(1);
#pragma unroll
  for (int j = 0; j < D; ++j) {
    p = add_rn(p, s[j]);
    beta = vmin(beta, mul_rn(p, T(1) / T(j + 1)));
  }
  beta = inside ? T(0) : beta;
  if constexpr (sizeof(T) == 4) {
    // z_k = clip(u_k -/+ beta): the sign of u_k - v_top (+0 on a tie: the
    // +1 block) moved onto beta >= 0 with one bit operation.
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const float d = u[k] - v_top;
      const float sb = __int_as_float(__float_as_int(beta) | (__float_as_int(d) & 0x80000000));
      z[k] = __saturatef(u[k] - sb);
    }
  } else {
    bool up[D];
#pragma unroll
    for (int k = 0; k < D; ++k) up[k] = u[k] >= v_top;
#pragma unroll
    for (int k = 0; k < D; ++k) z[k] = clip01(up[k] ? sub_rn(u[k], beta) : add_rn(u[k], beta));
  }
}

}  // namespace admm
