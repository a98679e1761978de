// Resident engine, regular-code fast path: every check has degree D and
// every variable degree DV (the (3,6) and (3,13) BASELINE codes).
//
// Same algorithm and frame scheduling as resident_decode_kernel
// (resident.cuh); what changes is how the work maps onto the SM:
//   * all degrees are compile-time, so the projection is branch-free
//     (project_pp_fixed) and no per-edge degree tests exist;
//   * every shared-memory address a thread touches in the hot loop -- the D
//     x-gather addresses of its checks, the DV message addresses of its
//     variables, its own message row and x slots -- is computed once per CTA
//     and kept in registers as a 32-bit shared address (bare LDS/STS);
//   * shared memory holds x[Npad] and the messages msg[D][Npad], the message
//     of edge (c, v) at msg[k][pi(v)] (k = the edge's slot in c, pi = the
//     internal variable numbering).  With the layout chosen by layout.h the
//     variable phase is bank-conflict-free by construction and the check
//     phase's x-gather / message store (both bank pi(v) mod 32) are spread
//     over the 32 banks (residual collisions reported by the optimiser);
//   * each thread owns VPT variables whose LLR/mu stays in registers;
//   * the stop rule runs as one barrier-reduction (__syncthreads_or): if any
//     thread's own partial residual sum already reaches eps^2 * E the frame
//     cannot have converged (sums of non-negative terms are monotone under
//     round-to-nearest), and the exact full sum is only formed when every
//     partial is below the threshold.
#pragma once

#include "resident.cuh"

namespace admm {

template <int D>
struct MsgStride {
  static constexpr int value = (D % 2 == 0) ? D + 1 : D;
};

// Padded variable count of the shared-memory arrays.  COL kernels also give
// every idle thread slot (variables i >= N, checks c >= M) real storage so the
// hot loop carries no activity predicates: idle variables occupy slots
// [N, VPT * NT) and idle checks gather from / write to the spare slot N.
__host__ __device__ constexpr bool regular_gm_smem(bool col, int minb, bool zs = false) { return col && minb >= 4 && !zs; }

__host__ __device__ inline int regular_np(int n_vars, bool col, int nt, int vpt) {
  if (!col) return (n_vars + 31) & ~31;
  const int need = (n_vars + 1 > vpt * nt ? n_vars + 1 : vpt * nt);
  return (need + 31) & ~31;
}

// NPC / NTC > 0 fix the padded variable count and the CTA size at compile
// time (COL only): every shared address in the hot loop is then a register
// plus an immediate offset.
// ZS keeps the edge state (z, lambda) in shared memory instead of registers
// (colored fp32 kernels): zs[q][j][NT] float4 {z_2j, z_2j+1, l_2j, l_2j+1},
// 16-byte accesses, conflict-free.  It buys registers for more resident warps
// where the register file, not shared memory, caps the CTAs per SM.
template <typename T, int D, int DV, int CPT, int VPT, int MINB, int MAXT = 512, bool COL = false, int NPC = 0,
          int NTC = 0, bool ZS = false>
__global__ void __launch_bounds__(MAXT, MINB) resident_regular_kernel(const ResidentParams<T> p,
                                                                     const int* __restrict__ var_edge) {
  static_assert(!COL || (D % DV <= 1 && VPT % 2 == 0), "colored layout: D mod DV in {0, 1}, VPT even");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int N = p.n_vars, M = p.n_checks;
  static_assert(COL || (NPC == 0 && NTC == 0), "compile-time geometry needs the colored layout");
  const int tid = threadIdx.x, NT = NTC ? NTC : blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nwarps = NT >> 5;
  const int NP = NPC ? NPC : COL ? regular_np(N, true, NT, VPT) : (N + 31) & ~31;
  constexpr int kRows = COL ? DV : D;  // message rows: colors (COL) or check slots
  static_assert(!ZS || (COL && D % 2 == 0), "shared-memory edge state: colored fp32 kernels");
  const int zs_bytes = ZS ? CPT * (D / 2) * NT * 16 : 0;
  const uint32_t zs_a = smem_u32(smem_raw) + 16u * tid;  // this thread's float4 column
  auto zsa = [&](int q, int j) -> uint32_t { return zs_a + 16u * ((q * (D / 2) + j) * NT); };
  T* xs = reinterpret_cast<T*>(smem_raw + zs_bytes);
  T* msg = xs + NP;
  // kGmSmem (colored kernels built for >= 4 CTAs/SM): the LLR steps gamma/mu
  // live in shared memory after the messages, read as pairs next to them --
  // four fewer registers (+1.5 % at 4 CTAs/SM; -3 % at one CTA per SM).
  constexpr bool kGmSmem = regular_gm_smem(COL, MINB, ZS);
  double* red = reinterpret_cast<double*>(msg + kRows * NP + (kGmSmem ? NP : 0));  // 8-byte aligned: NP % 32 == 0
  int* s_int = reinterpret_cast<int*>(red + 64);  // [0] frame, [1] weight
  const uint32_t msg_a = smem_u32(msg), xs_a = smem_u32(xs);
  constexpr uint32_t ES = sizeof(T);
  // msg[k][pi(v)] sits at x-address of v + moff(k)
  const uint32_t moff0 = NPC ? ES * NPC : msg_a - xs_a, mstride = ES * NP;
  // kRot: colored layout with D = q DV + 1 (the (3,13) code): slot k of a
  // check with rotation r has color (k + r) mod DV, so each check keeps its
  // DV color offsets in registers (rot_off).
  constexpr bool kRot = COL && (D % DV != 0);
  uint32_t rot_off[CPT][kRot ? DV : 1];
  // shared-address offset of the message of slot k of check q from the x slot of its variable
  auto moff = [&](int q, int k) -> uint32_t {
    if constexpr (kRot) return rot_off[q][k % DV];
    else return moff0 + (COL ? k % DV : k) * mstride;
  };

  // ---- per-thread graph registers (once per CTA) ----
  uint32_t xaddr[CPT][D];
  bool cact[CPT];
#pragma unroll
  for (int q = 0; q < CPT; ++q) {
    const int c = tid + q * NT;
    cact[q] = c < M;
    if constexpr (kRot) {
      const int r = cact[q] && p.check_rot ? __ldg(p.check_rot + c) : 0;
#pragma unroll
      for (int j = 0; j < DV; ++j) rot_off[q][j] = moff0 + ((j + r) % DV) * mstride;
    }
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const int v = cact[q] ? __ldg(p.chk_var + k * p.m_pad + c) : (COL ? N : 0);  // internal variable
      xaddr[q][k] = xs_a + ES * v;
    }
  }
  uint32_t vaddr[COL ? 1 : VPT][DV];
  uint32_t xst[VPT];
  int vorig[VPT];  // original variable of each owned internal variable (layout.h relabeling)
  bool vact[VPT];
#pragma unroll
  for (int q = 0; q < VPT; ++q) {
    // COL: variables in adjacent pairs (2 tid + 2 NT p, +1) so the variable
    // phase moves two of them per 8-byte shared access
    const int i = COL ? 2 * tid + 2 * NT * (q >> 1) + (q & 1) : tid + q * NT;
    vact[q] = i < N;
    if constexpr (!COL) {
#pragma unroll
      for (int j = 0; j < DV; ++j) {
        const int e = vact[q] ? __ldg(var_edge + i * DV + j) : 0;  // internal edge c * D + k
        vaddr[q][j] = msg_a + ES * ((e % D) * NP + i);
      }
    }
    xst[q] = COL ? xs_a + ES * 2 * tid + ES * (2 * NT * (q >> 1) + (q & 1)) : xs_a + ES * tid + ES * q * NT;
    vorig[q] = (vact[q] && p.var_orig) ? __ldg(p.var_orig + i) : i;
  }

  constexpr bool kF64 = sizeof(T) == 8;
  // Duals are kept SCALED, l = lambda / mu (the reference's message-passing
  // form, tests/test_admm.py:208-240): v = w + l, l' = l + (w - z'),
  // message = z' - l'.  No division or multiply by mu in the loop; lambda
  // is converted only at the state I/O boundary.
  constexpr bool kPacked = !kF64 && (D % 2 == 0);
  // fp32 keeps the state as packed edge pairs (kPacked) so the loop-carried
  // registers are the FFMA2/FADD2 operand pairs themselves.
  T z[kPacked ? 1 : CPT][D], lam[kPacked ? 1 : CPT][D];
  float2 zp[ZS ? 1 : CPT][kPacked && !ZS ? D / 2 : 1], lp[ZS ? 1 : CPT][kPacked && !ZS ? D / 2 : 1];
  auto zget = [&](int q, int k) -> T {
    if constexpr (ZS) {
      const float4 v = lds4(zsa(q, k >> 1));
      return (k & 1) ? v.y : v.x;
    } else if constexpr (kPacked) {
      return (k & 1) ? zp[q][k >> 1].y : zp[q][k >> 1].x;
    } else {
      return z[q][k];
    }
  };
  auto lget = [&](int q, int k) -> T {
    if constexpr (ZS) {
      const float4 v = lds4(zsa(q, k >> 1));
      return (k & 1) ? v.w : v.z;
    } else if constexpr (kPacked) {
      return (k & 1) ? lp[q][k >> 1].y : lp[q][k >> 1].x;
    } else {
      return lam[q][k];
    }
  };
  T gm[kGmSmem ? 1 : VPT];
  const float2 rho2 = make_float2(float(p.rho), float(p.rho));
  const float2 omr2 = make_float2(float(p.one_minus_rho), float(p.one_minus_rho));

  if (COL && tid == 0) sts(xs_a + ES * N, T(0));  // spare slot (no thread owns it when N == VPT * NT)
  for (;;) {
    __syncthreads();
    if (tid == 0) {
      s_int[0] = atomicAdd(p.queue, 1);
      s_int[1] = 0;
      if (!kF64) *reinterpret_cast<uint4*>(reinterpret_cast<uint32_t*>(red) + 4) = make_uint4(0, 0, 0, 0);  // t = 1
    }
    __syncthreads();
    const long long f = s_int[0];
    if (f >= p.batch) break;

    // ---- frame setup ----
#pragma unroll
    for (int q = 0; q < VPT; ++q) {
      const T g = vact[q] ? div_rn(frame_llr<T>(p, f, vorig[q]), p.mu) : T(0);
      if constexpr (kGmSmem) sts(xst[q] + moff0 + DV * mstride, g);
      else gm[q] = g;
    }
#pragma unroll
    for (int q = 0; q < CPT; ++q) {
      const int c = tid + q * NT;
#pragma unroll
      for (int k = 0; k < D; ++k) {
        T z0 = T(0), l0 = T(0);
        if (p.z_in != nullptr && cact[q]) {
          const long long e = f * p.ld_edge + (p.edge_ref ? __ldg(p.edge_ref + c * D + k) : c * D + k);
          z0 = p.z_in[e];
          l0 = p.lam_in[e];
        }
        const T s0 = div_rn(l0, p.mu);
        if constexpr (ZS) {
          // pairs are written once both halves are known
          if (k & 1) {
            zp[0][0].y = z0;
            lp[0][0].y = s0;
            sts4(zsa(q, k >> 1), make_float4(zp[0][0].x, z0, lp[0][0].x, s0));
          } else {
            zp[0][0].x = z0;
            lp[0][0].x = s0;
          }
        } else if constexpr (kPacked) {
          if (k & 1) {
            zp[q][k >> 1].y = z0;
            lp[q][k >> 1].y = s0;
          } else {
            zp[q][k >> 1].x = z0;
            lp[q][k >> 1].x = s0;
          }
        } else {
          z[q][k] = z0;
          lam[q][k] = s0;
        }
        // (COL: idle checks zero the spare slot's messages, so its x stays 0)
        if (COL || cact[q]) sts(xaddr[q][k] + moff(q, k), sub_rn(z0, s0));
      }
    }
    __syncthreads();

    int t = 0;
    bool converged = false;
    while (t < p.t_max) {
      ++t;
      // ---- x-update (admm_decoder.py:108-124): edges summed in edge order ----
      if constexpr (COL && kF64) {
        // fp64: pairs of variables in 16-byte accesses, messages summed in
        // color order (the reference sums in edge order; the difference is
        // at rounding level, inside the 1e-9 fp64 parity bar)
#pragma unroll
        for (int h = 0; h < VPT / 2; ++h) {
          const uint32_t a = xst[2 * h];
          double2 acc = lds2d(a + moff0);
#pragma unroll
          for (int j = 1; j < DV; ++j) {
            const double2 m = lds2d(a + moff0 + j * mstride);
            acc.x = add_rn(acc.x, m.x);
            acc.y = add_rn(acc.y, m.y);
          }
          const double inv = 1.0 / DV;
          sts2d(a, make_double2(clip01(mul_rn(sub_rn(acc.x, gm[2 * h]), inv)),
                                clip01(mul_rn(sub_rn(acc.y, gm[2 * h + 1]), inv))));
        }
      } else if constexpr (COL) {
        // pairs of variables: 8-byte loads/stores, packed sums (color order)
#pragma unroll
        for (int h = 0; h < VPT / 2; ++h) {
          const uint32_t a = xst[2 * h];
          float2 acc = lds2(a + moff0);
#pragma unroll
          for (int j = 1; j < DV; ++j) acc = __fadd2_rn(acc, lds2(a + moff0 + j * mstride));
          const float2 gm2 = kGmSmem ? lds2(a + moff0 + DV * mstride) : make_float2(gm[kGmSmem ? 0 : 2 * h], gm[kGmSmem ? 0 : 2 * h + 1]);
          const float2 num = fsub2_rn(acc, gm2);
          sts2(a, make_float2(clip01(num.x * (1.f / DV)), clip01(num.y * (1.f / DV))));
        }
      }
#pragma unroll
      for (int q = 0; q < (COL ? 0 : VPT); ++q) {
        if (COL || vact[q]) {
          // COL: message of color j at a fixed offset from the variable's x slot
          auto va = [&](int j) -> uint32_t { return COL ? xst[q] + moff0 + j * mstride : vaddr[COL ? 0 : q][j]; };
          T acc = lds(va(0), T());
#pragma unroll
          for (int j = 1; j < DV; ++j) acc = add_rn(acc, lds(va(j), T()));
          const T num = sub_rn(acc, gm[kGmSmem ? 0 : q]);
          const T xv = clip01(mul_rn(num, T(1) / T(DV)));  // reciprocal of the degree (compile time)
          sts(xst[q], xv);
        }
      }
      ADMM_JITTER();
      __syncthreads();
      // (fp32 stop-rule sums: buffer (t + 1) & 1 was last read in iteration
      // t - 1, which every thread left before this barrier)
      if (!kF64 && tid == 0) *reinterpret_cast<uint4*>(reinterpret_cast<uint32_t*>(red) + 4 * ((t + 1) & 1)) = make_uint4(0, 0, 0, 0);

      // ---- fused z-update, projection, residuals, lambda-update ----
      T primal = T(0), moved = T(0);
      if constexpr (kPacked) {
        // fp32: the elementwise updates run on packed pairs of edges (k, k+1)
        // with FFMA2/FADD2/FMUL2 -- same IEEE operations per lane, half the
        // instructions; the two residual sums are kept per lane and added at
        // the end (fp32 is the throughput mode, its summation order is free).
        float2 pr2 = make_float2(0.f, 0.f), mv2 = make_float2(0.f, 0.f);
#pragma unroll
        for (int q = 0; q < CPT; ++q) {
          // COL: idle checks run on the spare slot N, whose x, z, l and messages
          // stay exactly 0 (u = 0 projects to 0), so their residuals are 0
          if (COL || cact[q]) {
            float2 gx2[D / 2], u2[D / 2], z2[D / 2], l2[D / 2];
#pragma unroll
            for (int j = 0; j < D / 2; ++j) {
              gx2[j] = make_float2(lds(xaddr[q][2 * j], T()), lds(xaddr[q][2 * j + 1], T()));
              if constexpr (ZS) {
                const float4 v = lds4(zsa(q, j));
                z2[j] = make_float2(v.x, v.y);
                l2[j] = make_float2(v.z, v.w);
              } else {
                z2[j] = zp[q][j];
                l2[j] = lp[q][j];
              }
            }
            T u[D], zn[D];
#pragma unroll
            for (int j = 0; j < D / 2; ++j) {
              u2[j] = __fadd2_rn(__ffma2_rn(rho2, gx2[j], __fmul2_rn(omr2, z2[j])), l2[j]);
              u[2 * j] = u2[j].x;
              u[2 * j + 1] = u2[j].y;
            }
            project_pp_fixed<T, D>(u, zn);
#pragma unroll
            for (int j = 0; j < D / 2; ++j) {
              const float2 zn2 = make_float2(zn[2 * j], zn[2 * j + 1]);
              const float2 r1 = fsub2_rn(gx2[j], zn2);
              const float2 r2 = fsub2_rn(zn2, z2[j]);
              pr2 = __ffma2_rn(r1, r1, pr2);
              mv2 = __ffma2_rn(r2, r2, mv2);
              // reassociated dual update l' = (w + l) - z' = u - z' (fp32
              // throughput mode): w and l are dead once u is formed
              const float2 ln = fsub2_rn(u2[j], zn2);
              const float2 m2 = fsub2_rn(zn2, ln);
              if constexpr (ZS) {
                sts4(zsa(q, j), make_float4(zn2.x, zn2.y, ln.x, ln.y));
              } else {
                lp[q][j] = ln;
                zp[q][j] = zn2;
              }
              sts(xaddr[q][2 * j] + moff(q, 2 * j), m2.x);
              sts(xaddr[q][2 * j + 1] + moff(q, 2 * j + 1), m2.y);
            }
          }
        }
        primal = pr2.x + pr2.y;
        moved = mv2.x + mv2.y;
      } else {
#pragma unroll
      for (int q = 0; q < CPT; ++q) {
        if (cact[q]) {
          T gx[D], w[D], u[D], zn[D];
#pragma unroll
          for (int k = 0; k < D; ++k) gx[k] = lds(xaddr[q][k], T());
#pragma unroll
          for (int k = 0; k < D; ++k) {
            w[k] = add_rn(mul_rn(p.rho, gx[k]), mul_rn(p.one_minus_rho, z[kPacked ? 0 : q][k]));
            u[k] = add_rn(w[k], lam[kPacked ? 0 : q][k]);
          }
          project_pp_fixed<T, D>(u, zn);
#pragma unroll
          for (int k = 0; k < D; ++k) {
            const T r1 = sub_rn(gx[k], zn[k]);
            const T r2 = sub_rn(zn[k], z[kPacked ? 0 : q][k]);
            primal = add_rn(primal, mul_rn(r1, r1));
            moved = add_rn(moved, mul_rn(r2, r2));
            if constexpr (kF64) {
              lam[kPacked ? 0 : q][k] = add_rn(lam[kPacked ? 0 : q][k], sub_rn(w[k], zn[k]));
            } else {
              // fp32 (throughput mode), as in the packed path: l' = (w + l) - z'
              // = u - z', so w is dead once u is formed (13 registers at d = 13)
              lam[kPacked ? 0 : q][k] = sub_rn(u[k], zn[k]);
            }
            z[kPacked ? 0 : q][k] = zn[k];
            sts(xaddr[q][k] + moff(q, k), sub_rn(zn[k], lam[kPacked ? 0 : q][k]));
          }
        }
      }
      }
      // ---- stop rule (admm_decoder.py:169,174-181) ----
      // (p.thr is eps^2 E rounded up to T: a partial >= thr is >= the fp64
      // threshold; the exact sums below are accumulated in fp64)
      ADMM_JITTER();
      if (__syncthreads_or(primal >= p.thr || moved >= p.thr)) continue;
      if constexpr (!kF64) {
        // fp32 (throughput mode): every partial is below thr, so each one is
        // a 42-bit fixed-point number {hi, lo} (21 bits each, truncated below
        // 2^-42 of the scaled threshold); integer sums are exact and
        // order-free -- one REDUX per word and warp, shared-memory atomics
        // across the warps -- where the fp64 butterfly cost half an iteration
        // (13 % of all samples on the 1.5 dB point, whose stuck frames pass
        // the per-thread test every iteration).
        uint32_t* fx = reinterpret_cast<uint32_t*>(red) + 4 * (t & 1);
        const float ps = primal * p.fx_scale, ms = moved * p.fx_scale;
        const uint32_t ph = __float2uint_rz(ps), mh = __float2uint_rz(ms);
        const uint32_t pl = __float2uint_rz((ps - __uint2float_rn(ph)) * 2097152.f);
        const uint32_t ml = __float2uint_rz((ms - __uint2float_rn(mh)) * 2097152.f);
        const uint32_t s0 = __reduce_add_sync(0xffffffffu, ph), s1 = __reduce_add_sync(0xffffffffu, pl);
        const uint32_t s2 = __reduce_add_sync(0xffffffffu, mh), s3 = __reduce_add_sync(0xffffffffu, ml);
        if (lane == 0) {
          atomicAdd(fx, s0);
          atomicAdd(fx + 1, s1);
          atomicAdd(fx + 2, s2);
          atomicAdd(fx + 3, s3);
        }
        __syncthreads();
        const volatile uint32_t* fv = fx;
        const unsigned long long a = (static_cast<unsigned long long>(fv[0]) << 21) + fv[1];
        const unsigned long long b = (static_cast<unsigned long long>(fv[2]) << 21) + fv[3];
        if (a < p.fx_thr && b < p.fx_thr) {
          converged = true;
          break;
        }
        continue;
      }
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
#pragma unroll
    for (int q = 0; q < VPT; ++q) {
      if (vact[q]) {
        const int i = vorig[q];
        const T xv = lds(xst[q], T());
        const bool h = xv > T(0.5);
        ones += h;
        integral &= vmin(fabs(xv), fabs(T(1) - xv)) <= T(1e-5);
        if (p.x_out) p.x_out[f * p.ld_x + i] = xv;
        if (p.hard_out) p.hard_out[f * p.ld_hard + i] = h;
      }
    }
    bool odd = false;
#pragma unroll
    for (int q = 0; q < CPT; ++q) {
      if (cact[q]) {
        const int c = tid + q * NT;
        int par = 0;
#pragma unroll
        for (int k = 0; k < D; ++k) par ^= (lds(xaddr[q][k], T()) > T(0.5));
        odd |= par;
        if (p.z_out) {
#pragma unroll
          for (int k = 0; k < D; ++k) {
            const long long e = f * p.ld_edge + (p.edge_ref ? __ldg(p.edge_ref + c * D + k) : c * D + k);
            p.z_out[e] = zget(q, k);
            p.lam_out[e] = mul_rn(p.mu, lget(q, k));
          }
        }
      }
    }
    ones = __reduce_add_sync(0xffffffffu, ones);
    if (lane == 0 && ones) atomicAdd(s_int + 1, ones);
    const int all_integral = __syncthreads_and(integral);
    const int any_odd = __syncthreads_or(odd);
    if (tid == 0) {
      if (p.iters_out) p.iters_out[f] = t;
      if (p.flags_out)
        p.flags_out[f] = (converged ? kFlagConverged : 0) | (all_integral ? kFlagIntegral : 0) |
                         (any_odd ? 0 : kFlagCodeword);
      if (p.weight_out) p.weight_out[f] = s_int[1];
    }
  }
}

// Shared memory of the regular kernel (bytes): x[Npad] | msg[rows][Npad] | red (64 fp64) | ints,
// rows = D (slot layout) or DV (colored layout).
inline int regular_smem_bytes(int elem, int D, int DV, int n_vars, bool col, bool gm_smem, int nt, int vpt,
                              int np_fixed = 0, int zs_cpt = 0) {
  const int np = np_fixed ? np_fixed : regular_np(n_vars, col, nt, vpt);
  return zs_cpt * (D / 2) * nt * 16 + elem * (np + (col ? DV : D) * np + (gm_smem ? np : 0)) + 8 * 64 + 16;
}

}  // namespace admm
