// Exact Euclidean projection onto the parity polytope PP_d, in registers.
//
// Contract: the reference's project_batch (parity_polytope.py:352-421), which
//   sorts v = u descending, takes r = 2 floor(sum clip(v) / 2)        :366-372
//   tests the facet f = +1 on the top r+1 coordinates, -1 elsewhere   :374-382
//   and otherwise returns z = clip(v - beta f, 0, 1) with beta the root of
//   g(beta) = f . clip(v - beta f, 0, 1) = r on [0, beta_max]         :385-414
// Writing s_k for the shift at which coordinate k enters the open band (0,1)
// -- s_k = u_k - 1 on the +1 block, -u_k on the -1 block -- every coordinate is
// active on exactly (s_k, s_k + 1), so g(beta) = (r + 1) - sum_k clip(beta -
// s_k, 0, 1) and the root solves sum_k max(beta - s_k, 0) = 1: water-filling.
// With s sorted ascending and P_j = 1 + s_(1) + ... + s_(j) every P_j / j
// over-estimates the root and the active prefix attains it.  The cut-search
// formulation below gets the block f, the sorted shifts and the facet test
// from ONE sorting network.  Results agree with project_batch to rounding
// (tests/test_gpu_projection.py against the reference's goldens,
// tests/test_projection_cut.py for the formulation itself).
//
// Degree handling: arrays are sized D (a compile-time bucket); the active
// degree d <= D is implied by the padding: slots k >= d must hold -inf in u.
#pragma once

#include "common.cuh"
#include "sortnet.cuh"

namespace admm {

// Sum of c[0..d) in numpy's pairwise_sum order for short rows: sequential
// below 8 elements, eight interleaved partial sums combined as a tree and a
// sequential tail otherwise.  Zeros in padded slots leave the sequential sum
// unchanged.  Used by the membership kernel (steps.cu), whose r = even floor
// of the l1 norm must match the reference bit for bit where the norm sits on
// an even integer.
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

// Project u (degree d <= D; u[k] = -inf for k >= d) onto PP_d; z[k] = 0 for
// k >= d.  Generic-degree kernels (resident.cuh, steps.cu, project.cu).
template <typename T, int D>
__device__ __forceinline__ void project_pp(const T (&u)[D], T (&z)[D], int /*d*/) {
  project_pp_cut<T, D>(u, z);
}

// Fixed-degree entry of the regular-code kernels (d == D at compile time).
template <typename T, int D>
__device__ __forceinline__ void project_pp_fixed(const T (&u)[D], T (&z)[D]) {
  project_pp_cut<T, D>(u, z);
}

}  // namespace admm
