// Cluster-resident engine: one thread-block CLUSTER decodes one frame, with
// the frame's state spread over the cluster's SMs (BASELINE config 5,
// n = 16384, m = 8192: 16 CTAs x 512 checks).
//
// It is the resident engine (resident_regular.cuh) stretched over a cluster:
//   * CTA r of C owns checks [r*MC, (r+1)*MC) and variables [r*NC, (r+1)*NC);
//     z and lambda of its checks' edges live in registers for the whole
//     decode, its checks' messages z - lambda/mu and its variables' x live in
//     its shared memory;
//   * the x-gather of a check and the message-gather of a variable read the
//     owning CTA's shared memory through DSMEM (ld.shared::cluster); every
//     such address is resolved once per CTA with mapa and kept in a register;
//   * the two __syncthreads of an iteration become cluster barriers
//     (barrier.cluster.arrive.release / wait.acquire);
//   * the stop rule: each CTA reduces "some partial >= eps^2 E" with one
//     __syncthreads_or and posts the flag to CTA 0; after the cluster barrier
//     every warp reads the C flags.  Only when no CTA is above the threshold
//     are the exact sums formed and exchanged the same way (fixed order, so
//     every thread of the cluster takes the same decision).
// The cluster is persistent and pulls frames from a global queue, exactly
// like the single-CTA resident engine.
#pragma once

#include "resident.cuh"
#include "resident_regular.cuh"

namespace admm {

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_size() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ float ldc(uint32_t a, float) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ double ldc(uint32_t a, double) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void stc(uint32_t a, float v) {
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}
__device__ __forceinline__ void stc(uint32_t a, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
__device__ __forceinline__ void stc_u32(uint32_t a, uint32_t v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ldc_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Per-CTA shared memory of the cluster kernel (bytes).
inline int cluster_smem_bytes(int elem, int D, int mc_pad, int nc) {
  const int ds = (D % 2 == 0) ? D + 1 : D;
  // msg rows | x | red(64 T) | exchange area: 16 flags, 32 sums (T), 16 ints x 4, frame
  return elem * (mc_pad * ds + ((nc + 1) & ~1) + 64 + 32) + 4 * (16 * 6 + 8) + 16;
}

template <typename T, int D, int DV, int CPT, int VPT>
__global__ void __launch_bounds__(512, 1) cluster_decode_kernel(const ResidentParams<T> p,
                                                                const int* __restrict__ var_edge, int MC, int NC) {
  constexpr int DS = MsgStride<D>::value;
  constexpr uint32_t ES = sizeof(T);
  constexpr bool kF64 = sizeof(T) == 8;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int N = p.n_vars, M = p.n_checks;
  const int tid = threadIdx.x, NT = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nwarps = NT >> 5;
  const uint32_t rank = cluster_rank(), C = cluster_size();
  const int mc_pad = NT * CPT;
  T* msg = reinterpret_cast<T*>(smem_raw);
  T* xs = msg + mc_pad * DS;
  T* red = xs + ((NC + 1) & ~1);
  T* xsum = red + 64;                                  // [16][2] exact sums posted to CTA 0
  int* xflag = reinterpret_cast<int*>(xsum + 32);      // [16] not-converged flags
  int* xint = xflag + 16;                              // [16] integral flags
  int* xodd = xint + 16;                               // [16] odd-parity flags
  int* xwt = xodd + 16;                                // [16] weights
  int* s_frame = xwt + 16;                             // [1]
  const uint32_t msg_a = smem_u32(msg), xs_a = smem_u32(xs);

  // ---- per-thread addresses (once per CTA) ----
  uint32_t xaddr[CPT][D];
  uint32_t mrow[CPT];
  bool cact[CPT];
#pragma unroll
  for (int q = 0; q < CPT; ++q) {
    const int lc = tid + q * NT, gc = rank * MC + lc;
    cact[q] = lc < MC && gc < M;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const int v = cact[q] ? __ldg(p.chk_var + k * p.m_pad + gc) : 0;
      const int owner = v / NC;
      xaddr[q][k] = mapa(xs_a + ES * (v - owner * NC), owner);
    }
    mrow[q] = msg_a + ES * (lc * DS);
  }
  uint32_t vaddr[VPT][DV];
  uint32_t xst[VPT];
  bool vact[VPT];
#pragma unroll
  for (int q = 0; q < VPT; ++q) {
    const int lv = tid + q * NT, gi = rank * NC + lv;
    vact[q] = lv < NC && gi < N;
#pragma unroll
    for (int j = 0; j < DV; ++j) {
      const int e = vact[q] ? __ldg(var_edge + gi * DV + j) : 0;
      const int c = e / D, k = e % D;
      const int owner = c / MC;
      vaddr[q][j] = mapa(msg_a + ES * ((c - owner * MC) * DS + k), owner);
    }
    xst[q] = xs_a + ES * lv;
  }
  // CTA 0's exchange area, seen from this CTA.
  const uint32_t flag0 = mapa(smem_u32(xflag), 0), sum0 = mapa(smem_u32(xsum), 0);
  const uint32_t int0 = mapa(smem_u32(xint), 0), odd0 = mapa(smem_u32(xodd), 0), wt0 = mapa(smem_u32(xwt), 0);

  const T inv_mu = p.inv_mu;
  T z[CPT][D], lam[CPT][D];
  T gm[VPT];
  cluster_barrier();  // every CTA of the cluster is running before any DSMEM access

  for (;;) {
    if (rank == 0 && tid == 0) {
      const int f = atomicAdd(p.queue, 1);
      for (uint32_t r = 0; r < C; ++r) stc_u32(mapa(smem_u32(s_frame), r), static_cast<uint32_t>(f));
    }
    cluster_barrier();
    const long long f = static_cast<int>(*reinterpret_cast<volatile int*>(s_frame));
    if (f >= p.batch) break;

    // ---- frame setup ----
#pragma unroll
    for (int q = 0; q < VPT; ++q)
      gm[q] = vact[q] ? div_rn(frame_llr<T>(p, f, rank * NC + tid + q * NT), p.mu) : T(0);
#pragma unroll
    for (int q = 0; q < CPT; ++q) {
#pragma unroll
      for (int k = 0; k < D; ++k) {
        z[q][k] = T(0);
        lam[q][k] = T(0);
        if (cact[q]) sts(mrow[q] + ES * k, T(0));
      }
    }
    cluster_barrier();

    int t = 0;
    bool converged = false;
    while (t < p.t_max) {
      ++t;
      // ---- x-update over this CTA's variables (messages via DSMEM) ----
#pragma unroll
      for (int q = 0; q < VPT; ++q) {
        if (vact[q]) {
          T mv[DV];
#pragma unroll
          for (int j = 0; j < DV; ++j) mv[j] = ldc(vaddr[q][j], T());
          T acc = mv[0];
#pragma unroll
          for (int j = 1; j < DV; ++j) acc = add_rn(acc, mv[j]);
          const T num = sub_rn(acc, gm[q]);
          sts(xst[q], clip01(mul_rn(num, T(1) / T(DV))));
        }
      }
      cluster_barrier();

      // ---- fused check update over this CTA's checks (x via DSMEM) ----
      T primal = T(0), moved = T(0);
#pragma unroll
      for (int q = 0; q < CPT; ++q) {
        if (cact[q]) {
          T gx[D], w[D], u[D], zn[D];
#pragma unroll
          for (int k = 0; k < D; ++k) gx[k] = ldc(xaddr[q][k], T());
#pragma unroll
          for (int k = 0; k < D; ++k) {
            w[k] = add_rn(mul_rn(p.rho, gx[k]), mul_rn(p.one_minus_rho, z[q][k]));
            u[k] = add_rn(w[k], lam[q][k]);  // scaled dual lambda/mu
          }
          project_pp_fixed<T, D>(u, zn);
#pragma unroll
          for (int k = 0; k < D; ++k) {
            const T r1 = sub_rn(gx[k], zn[k]);
            const T r2 = sub_rn(zn[k], z[q][k]);
            primal = add_rn(primal, mul_rn(r1, r1));
            moved = add_rn(moved, mul_rn(r2, r2));
            lam[q][k] = add_rn(lam[q][k], sub_rn(w[k], zn[k]));
            z[q][k] = zn[k];
            sts(mrow[q] + ES * k, sub_rn(zn[k], lam[q][k]));
          }
        }
      }
      // ---- stop rule (admm_decoder.py:169,174-181), cluster-wide ----
      const int above = __syncthreads_or(primal >= p.thr || moved >= p.thr);
      if (tid == 0) stc_u32(flag0 + 4 * rank, static_cast<uint32_t>(above));
      cluster_barrier();
      const uint32_t fl = lane < static_cast<int>(C) ? ldc_u32(flag0 + 4 * lane) : 0u;
      if (__any_sync(0xffffffffu, fl != 0)) continue;
      // every partial is below the threshold: exact sums, fixed order
      primal = warp_allsum(primal);
      moved = warp_allsum(moved);
      if (lane == 0) {
        red[2 * warp] = primal;
        red[2 * warp + 1] = moved;
      }
      __syncthreads();
      T a = lane < nwarps ? red[2 * lane] : T(0);
      T b = lane < nwarps ? red[2 * lane + 1] : T(0);
      a = warp_allsum(a);
      b = warp_allsum(b);
      if (tid == 0) {
        stc(sum0 + ES * (2 * rank), a);
        stc(sum0 + ES * (2 * rank + 1), b);
      }
      cluster_barrier();
      a = lane < static_cast<int>(C) ? ldc(sum0 + ES * (2 * lane), T()) : T(0);
      b = lane < static_cast<int>(C) ? ldc(sum0 + ES * (2 * lane + 1), T()) : T(0);
      a = warp_allsum(a);
      b = warp_allsum(b);
      cluster_barrier();  // everyone has read the sums before they can be rewritten
      if (a < p.thr && b < p.thr) {
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
        const int i = rank * NC + tid + q * NT;
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
        int par = 0;
#pragma unroll
        for (int k = 0; k < D; ++k) par ^= (ldc(xaddr[q][k], T()) > T(0.5));
        odd |= par;
      }
    }
    ones = __reduce_add_sync(0xffffffffu, ones);
    if (lane == 0) red[warp] = T(ones);
    const int all_int = __syncthreads_and(integral);
    const int any_odd = __syncthreads_or(odd);
    if (tid == 0) {
      int wsum = 0;
      for (int q = 0; q < nwarps; ++q) wsum += static_cast<int>(red[q]);
      stc_u32(int0 + 4 * rank, static_cast<uint32_t>(all_int));
      stc_u32(odd0 + 4 * rank, static_cast<uint32_t>(any_odd));
      stc_u32(wt0 + 4 * rank, static_cast<uint32_t>(wsum));
    }
    cluster_barrier();
    if (rank == 0 && tid == 0) {
      int ai = 1, ao = 0, w = 0;
      for (uint32_t r = 0; r < C; ++r) {
        ai &= xint[r] != 0;
        ao |= xodd[r] != 0;
        w += xwt[r];
      }
      if (p.iters_out) p.iters_out[f] = t;
      if (p.flags_out)
        p.flags_out[f] = (converged ? kFlagConverged : 0) | (ai ? kFlagIntegral : 0) | (ao ? 0 : kFlagCodeword);
      if (p.weight_out) p.weight_out[f] = w;
    }
    cluster_barrier();  // exchange area and s_frame free for the next frame
  }
}

}  // namespace admm
