// Cluster engine: one thread-block CLUSTER of C CTAs decodes one frame of a
// code too large for one SM (BASELINE config 5, n = 16384: C = 4 CTAs of
// 1024 threads, one per SM), with every byte of the frame's decoder state on
// chip.  fp32 (throughput mode): C = 8 CTAs of 512 threads, two per SM (or
// C = 4 of 1024); fp64 (parity mode): C = 8 CTAs of 512 threads at 128
// registers, one per SM -- the reference's expression tree per edge
// (resident_regular.cuh's fp64 path), state twice the size.
//
// Layout (cluster_layout.h): CTA p owns M/C checks and N/C variables; the
// variables its checks touch but other CTAs own are GHOSTS with local slots.
// Per CTA and iteration, exactly the resident kernel's work
// (resident_regular.cuh, colored layout, packed fp32 pairs) plus two
// table-driven exchanges over DSMEM, each a warp-coalesced copy into
// CONSECUTIVE words of the destination (~20-25 B/cycle; scattered 4-byte
// remote accesses cost ~2.6 cycles each, tools/micro/dsmem.cu):
//
//   variable    x = clip((sum_j msg_j - gamma/mu) / DV) of own variables
//   x-send      own x -> ghost slots of the CTAs holding them  (DSMEM)
//   -- cluster barrier A --
//   check       gather x (own + ghost slots), project, dual update, message
//               to msg[color][slot(v)] (own rows, or ghost rows)
//   msg-send    ghost-row messages -> the owners' message rows  (DSMEM)
//               stop-rule header {flag, exact sums} -> every CTA
//   -- cluster barrier B --
//   decision    every thread reads the C headers: uniform, deterministic
//
// Stop rule (admm_decoder.py:169,174-181): each CTA forms its partials as the
// resident kernel does; when no partial reaches eps^2 E it also forms the
// CTA's exact sums in fp64; the frame converged iff every CTA's flag is clear
// and the fp64 sum of the C CTA sums (rank order) is below the threshold.
// Frames are pulled from a global queue by CTA 0 and broadcast to the
// cluster; the outputs (make_output, is_codeword) are reduced into CTA 0.
#pragma once

#include "resident_regular.cuh"
#include "synth.cuh"

namespace admm {

constexpr int kClusterMax = 8;

// Packed exchange-table entries (cluster_layout.h / abi.cu):
//   x-send   own slot (13 bits) | ghost slot in the destination (16) << 13 | rank (3) << 29
//   msg-send color (2) | ghost slot here (13) << 2 | own slot at the owner (12) << 15 | owner (3) << 27
//            (cluster_layout.h ms_entry)
__host__ __device__ constexpr uint32_t xs_pack(uint32_t src, uint32_t dst, uint32_t r) { return src | dst << 13 | r << 29; }

__device__ __forceinline__ uint32_t cl_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cl_mapa(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
// DSMEM address of local shared address `a` in CTA `rank` (checked build:
// `a` inside the shared window, rank inside the cluster).
template <int C>
__device__ __forceinline__ uint32_t cl_addr(uint32_t a, uint32_t rank, uint32_t bytes = 4) {
  ADMM_CHECK_SMEM(a, bytes);
  ADMM_ASSERT(rank < static_cast<uint32_t>(C));
  return cl_mapa(a, rank);
}
__device__ __forceinline__ void cl_st(uint32_t a, float v) {
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}
__device__ __forceinline__ void cl_st_u32(uint32_t a, uint32_t v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void cl_st_f64(uint32_t a, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
// st.async: non-blocking DSMEM store whose completion releases tx bytes on the
// destination CTA's mbarrier `mb` (shared::cluster address).
__device__ __forceinline__ void cl_st_async(uint32_t a, float v, uint32_t mb) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(a),
               "r"(__float_as_uint(v)), "r"(mb)
               : "memory");
}
__device__ __forceinline__ void cl_st_async(uint32_t a, double v, uint32_t mb) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(a),
               "l"(__double_as_longlong(v)), "r"(mb)
               : "memory");
}
__device__ __forceinline__ void cl_st(uint32_t a, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
__device__ __forceinline__ void cl_st_async_u32(uint32_t a, uint32_t v, uint32_t mb) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(a), "r"(v), "r"(mb)
               : "memory");
}
__device__ __forceinline__ void cl_st_async_f64(uint32_t a, double v, uint32_t mb) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(a),
               "l"(__double_as_longlong(v)), "r"(mb)
               : "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t mb, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mb), "r"(count) : "memory");
}
// One arrival that also expects `bytes` of transactions in the current phase.
__device__ __forceinline__ void mbar_expect(uint32_t mb, uint32_t bytes) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(mb),
               "r"(bytes)
               : "memory");
}
// Wait for the phase with parity `par` to complete (acquire); a wait that never
// completes traps after ~2^26 tries instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint32_t mb, uint32_t par) {
  for (uint32_t k = 0;; ++k) {
    uint32_t done;
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(mb), "r"(par)
        : "memory");
    if (done) return;
    if (k > (1u << 26)) {
      printf("ADMM: cluster mbarrier wait timed out (block %d thread %d)\n", blockIdx.x, threadIdx.x);
      __trap();
    }
  }
}
__device__ __forceinline__ void cl_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// CTA-rank bits of a shared::cluster address (checked at kernel start)
constexpr uint32_t kCtaBits = 0xff000000u;  // (the top byte: exchange() splices it with PRMT)
__device__ __forceinline__ uint2 lds2u(uint32_t a) {
  ADMM_CHECK_SMEM(a, 8);
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ uint4 lds4u(uint32_t a) {
  ADMM_CHECK_SMEM(a, 16);
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts4u(uint32_t a, uint32_t v) {  // four words of v
  ADMM_CHECK_SMEM(a, 16);
  asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void sts2u(uint32_t a, uint32_t x, uint32_t y) {
  ADMM_CHECK_SMEM(a, 8);
  asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(a), "r"(x), "r"(y) : "memory");
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}

template <typename T>
struct ClusterParamsT {
  // graph (cluster_layout.h), per-part arrays flattened [C][...]
  const int* chk_slot;   // [C][D][MC]
  const int* chk_orig;   // [C][MC] original check (-1: idle slot)
  const int* own_var;    // [C][NO]
  const uint32_t* xsend; // [C][NXS] xs_pack(own slot, ghost slot, rank)
  const uint32_t* msend; // [C][NMS] ms_entry(color, ghost slot, owner's own slot, owner)
  int NPL, NXS, NMS, MC, NO;
  int sm_xs, sm_ms, sm_hdr, sm_mbar, sm_misc;  // ClusterSmem offsets (host-computed: constant-bank operands)
  int n_xs[kClusterMax], n_ms[kClusterMax];
  uint32_t rx_x[kClusterMax], rx_m[kClusterMax];  // MBAR: bytes each CTA receives per iteration
  // every CTA ships ghost x to every other CTA: the point-to-point (MBAR)
  // syncs then order every pair of CTAs within one iteration (see the kernel)
  int dense;
  int n_vars, n_checks;
  // frames
  long long batch;
  const T* gamma;
  long long ld_gamma;
  T mu, rho, one_minus_rho, thr;  // thr: eps^2 E rounded up to T (early-out)
  double thr_d;                   // eps^2 E
  float fx_scale;                 // fp32: 42-bit fixed-point stop-rule sums (ResidentParams::fx_scale)
  unsigned long long fx_thr;
  int t_max;
  T* x_out;
  long long ld_x;
  uint8_t* hard_out;
  long long ld_hard;
  int* iters_out;
  uint8_t* flags_out;
  int* weight_out;
  int* queue;
  SynthParams synth;
};
using ClusterParams = ClusterParamsT<float>;

// Shared memory (bytes): X | MSG[DV] | GM (each NPL elements) | xsend[NXS] |
// msend[NMS] (8-byte pre-mapped entries, below) | header | mbarriers | misc.
// Stop-rule header one CTA sends to every CTA each iteration: its exact fp64
// sums (valid when its flag is clear) and its "some partial >= threshold" flag.
// Structure of arrays, so the C flags every thread reads each iteration are
// two 16-byte loads.
struct ClusterHeader {
  double primal[kClusterMax], moved[kClusterMax];
  uint32_t flag[kClusterMax];
};

struct ClusterSmem {
  int x, xs, ms, hdr, mbar, misc, total;
  __host__ __device__ ClusterSmem(int elem, int NPL, int DV, int NXS, int NMS) {
    x = 0;
    xs = elem * NPL * (DV + 2);
    ms = xs + 8 * NXS;
    hdr = (ms + 8 * NMS + 15) & ~15;   // [2 parities] ClusterHeader
    mbar = hdr + 2 * static_cast<int>(sizeof(ClusterHeader));  // two mbarriers (x, messages)
    misc = mbar + 16;                    // ints: frame, weight + per-CTA output slots
    total = misc + 4 * (8 + 3 * kClusterMax) + 64 * 8;  // + fp64 block-reduction slots
  }
};

// Phase profiler (admm_cluster_phase_profile; the PROF instantiation): thread
// 0 of CTA 0 accumulates clock64() per phase: {-, variable, x-send,
// barrier A, check, msg-send, barrier B + decision, iterations}.
__device__ unsigned long long g_cl_cycles[8];

// MBAR (default when p.dense): the two per-iteration syncs are point-to-point:
// every remote store is an st.async that completes tx bytes on the
// destination's mbarrier, and a CTA waits only for the bytes it receives
// (ghost x; messages + every CTA's header) instead of an all-to-all cluster
// barrier (333 -> 354 G edge-updates/s on config 5).  Why no store can land
// in a buffer or an mbarrier phase still in use:
//   * o's x-send of iteration t+1 into q follows o's message wait of t, which
//     needs q's header of t, which q sends after its check phase of t (the
//     last reader of its ghost x of t, and after q's x-wait of t completed);
//   * q's msg-send of t+1 into o follows q's x-wait of t+1, which needs o's
//     x-send of t+1 (dense: every CTA ships x to every other), which follows
//     o's variable phase of t+1 (the last reader of its message rows of t)
//     and o's message wait of t;
//   * headers alternate between two buffers by iteration parity, and the
//     same chains keep every pair of CTAs within one iteration.
template <typename T, int D, int DV, int CPT, int VPT, int C, int NT, bool PROF = false, bool MBAR = false, int NPLC = 0>
__global__ void __cluster_dims__(C, 1, 1) __launch_bounds__(NT, (sizeof(T) == 4 ? 1024 : 512) / NT)
    cluster_decode_kernel(const ClusterParamsT<T> p) {
  static_assert(D % DV == 0 && D % 2 == 0 && VPT % 2 == 0, "cluster engine: colored layout");
  constexpr uint32_t ES = sizeof(T);
  constexpr bool kF64 = ES == 8;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int NPL = NPLC ? NPLC : p.NPL;  // NPLC: compile-time slot count (message rows at immediate offsets)
  const uint32_t rank = cl_rank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int nwarps = NT / 32;
  const uint32_t xs_a = smem_u32(smem_raw);  // X[NPL]; MSG[j] at +ES NPL (j + 1); GM at +ES NPL (DV + 1)
  const uint32_t mstride = ES * NPL;
  ClusterHeader* hdr = reinterpret_cast<ClusterHeader*>(smem_raw + p.sm_hdr);  // [2 parities]
  const uint32_t mb_x = smem_u32(smem_raw + p.sm_mbar), mb_m = mb_x + 8;        // mbarriers (MBAR)
  int* misc = reinterpret_cast<int*>(smem_raw + p.sm_misc);                     // [0] frame [1] weight
  int* outslot = misc + 8;                                                   // [C][3] integral, weight, odd
  double* red = reinterpret_cast<double*>(smem_raw + p.sm_misc + 4 * (8 + 3 * kClusterMax));

  // ---- per-part exchange tables into shared memory (once per CTA), pre-mapped:
  // 8-byte entries {DSMEM destination address, local source address} (the
  // order st.async wants its {address, mbarrier} register pair in), so an
  // exchange costs per entry one LDS.64, the source LDS, one LOP3 (the
  // destination's mbarrier: same CTA bits, fixed offset) and the st.async ----
  const uint32_t tx_b = smem_u32(smem_raw) + p.sm_xs, tm_b = smem_u32(smem_raw) + p.sm_ms;
  const uint32_t tx_a = tx_b + 8u * tid, tm_a = tm_b + 8u * tid;
  {
    const uint32_t* gx = p.xsend + static_cast<size_t>(rank) * p.NXS;
    const uint32_t* gms = p.msend + static_cast<size_t>(rank) * p.NMS;
    for (int i = tid; i < p.n_xs[rank]; i += NT) {
      const uint32_t u = __ldg(gx + i);
      sts2u(tx_a + 8u * (i - tid), cl_addr<C>(xs_a + ES * ((u >> 13) & 0xffffu), u >> 29, ES),
            xs_a + ES * (u & 0x1fffu));
    }
    for (int i = tid; i < p.n_ms[rank]; i += NT) {
      const uint32_t u = __ldg(gms + i);
      const uint32_t row = mstride * ((u & 3u) + 1);
      sts2u(tm_a + 8u * (i - tid), cl_addr<C>(xs_a + row + ES * ((u >> 15) & 0xfffu), u >> 27, ES),
            xs_a + row + ES * ((u >> 2) & 0x1fffu));
    }
    // shared::cluster addresses keep the CTA in the bits above the offset (a
    // CTA's own shared addresses carry its own): a destination's mbarrier is
    // (dst & kCtaBits) | (own mbarrier & ~kCtaBits)
    if (tid < C) {
      const uint32_t m = cl_mapa(mb_x, tid), a = cl_mapa(xs_a, tid);
      if (((m ^ mb_x) & ~kCtaBits) != 0 || ((a ^ xs_a) & ~kCtaBits) != 0 || (m & kCtaBits) != (a & kCtaBits)) {
        printf("ADMM: unexpected shared::cluster address layout (%x -> %x, %x -> %x)\n", mb_x, m, xs_a, a);
        __trap();
      }
    }
  }

  // ---- per-thread graph registers: checks lc = tid + q NT, own variable
  // pairs (2 tid + 2 NT h, +1) ----
  uint32_t xaddr[CPT][D];
  uint32_t cmask = 0;  // bit q: check q active
#pragma unroll
  for (int q = 0; q < CPT; ++q) {
    const int lc = tid + q * NT;
    if (__ldg(p.chk_orig + static_cast<size_t>(rank) * p.MC + lc) >= 0) cmask |= 1u << q;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const int s = __ldg(p.chk_slot + (static_cast<size_t>(rank) * D + k) * p.MC + lc);
      xaddr[q][k] = xs_a + ES * s;
    }
  }
  // own slots: xst(q) = xs0 + ES (2 NT (q >> 1) + (q & 1)) (compile-time offsets)
  const uint32_t xs0 = xs_a + 2u * ES * tid;
  const int* own_var = p.own_var + static_cast<size_t>(rank) * p.NO;
  auto xst = [&](int q) -> uint32_t { return xs0 + ES * (2 * NT * (q >> 1) + (q & 1)); };
  auto vorig = [&](int q) -> int { return __ldg(own_var + 2 * tid + 2 * NT * (q >> 1) + (q & 1)); };

  // edge state in registers: packed fp32 pairs, or the fp64 replicas and scaled duals
  const float2 rho2 = make_float2(float(p.rho), float(p.rho));
  const float2 omr2 = make_float2(float(p.one_minus_rho), float(p.one_minus_rho));
  float2 zp[kF64 ? 1 : CPT][kF64 ? 1 : D / 2], lp[kF64 ? 1 : CPT][kF64 ? 1 : D / 2];
  double zd[kF64 ? CPT : 1][kF64 ? D : 1], ld[kF64 ? CPT : 1][kF64 ? D : 1];
  const bool prof = PROF && blockIdx.x == 0 && tid == 0;
  long long tp = 0;
  auto phase = [&](int k) {
    if (prof) {
      const long long t2 = clock64();
      g_cl_cycles[k] += t2 - tp;
      tp = t2;
    }
  };

  // one table-driven exchange: entry i of this CTA's table (at tb + 8 i) is
  // handled by thread i mod NT
  auto exchange = [&](uint32_t tb, int n, uint32_t mb) {
    const uint32_t end = tb + 8u * n;
    for (uint32_t a = tb + 8u * tid; a < end; a += 8u * NT) {
      const uint2 e = lds2u(a);  // {destination, source}
      const T v = lds(e.y, T());
      if constexpr (MBAR)  // the destination's mbarrier: its CTA byte over our mbarrier's offset (one PRMT)
        cl_st_async(e.x, v, __byte_perm(mb, e.x, 0x7210));
      else
        cl_st(e.x, v);
    }
  };
  // x-update of own pair h (admm_decoder.py:108-124; colors summed in order)
  auto var_pair = [&](int h) {
    const uint32_t a = xst(2 * h);
    if constexpr (kF64) {
      // fp64: the resident fp64 kernel's variable update (16-byte pairs, colors
      // summed in order, times the reciprocal degree)
      double2 acc = lds2d(a + mstride);
#pragma unroll
      for (int j = 1; j < DV; ++j) {
        const double2 m = lds2d(a + mstride * (j + 1));
        acc.x = add_rn(acc.x, m.x);
        acc.y = add_rn(acc.y, m.y);
      }
      const double2 gm = lds2d(a + mstride * (DV + 1));
      const double inv = 1.0 / DV;
      sts2d(a, make_double2(clip01(mul_rn(sub_rn(acc.x, gm.x), inv)), clip01(mul_rn(sub_rn(acc.y, gm.y), inv))));
    } else {
      float2 acc = lds2(a + mstride);
#pragma unroll
      for (int j = 1; j < DV; ++j) acc = __fadd2_rn(acc, lds2(a + mstride * (j + 1)));
      const float2 num = fsub2_rn(acc, lds2(a + mstride * (DV + 1)));
      sts2(a, make_float2(clip01(num.x * (1.f / DV)), clip01(num.y * (1.f / DV))));
    }
  };
  // fused z-update, projection, residuals, dual update of check q: packed fp32
  // pairs, or (fp64) the reference's expression tree edge by edge
  // (admm_decoder.py:127-149 in the scaled-dual form of resident_regular.cuh)
  float2 pr2, mv2;
  double prd = 0.0, mvd = 0.0;
  auto check = [&](int q) {
    if constexpr (kF64) {
      double gx[D], w[D], u[D], zn[D];
#pragma unroll
      for (int k = 0; k < D; ++k) gx[k] = lds(xaddr[q][k], double());
#pragma unroll
      for (int k = 0; k < D; ++k) {
        w[k] = add_rn(mul_rn(p.rho, gx[k]), mul_rn(p.one_minus_rho, zd[q][k]));
        u[k] = add_rn(w[k], ld[q][k]);
      }
      project_pp_fixed<double, D>(u, zn);
#pragma unroll
      for (int k = 0; k < D; ++k) {
        const double r1 = sub_rn(gx[k], zn[k]);
        const double r2 = sub_rn(zn[k], zd[q][k]);
        prd = add_rn(prd, mul_rn(r1, r1));
        mvd = add_rn(mvd, mul_rn(r2, r2));
        ld[q][k] = add_rn(ld[q][k], sub_rn(w[k], zn[k]));
        zd[q][k] = zn[k];
        sts(xaddr[q][k] + mstride * (1 + k % DV), sub_rn(zn[k], ld[q][k]));
      }
    } else {
    float2 gx2[D / 2], u2[D / 2];
#pragma unroll
    for (int j = 0; j < D / 2; ++j) gx2[j] = make_float2(lds(xaddr[q][2 * j], 0.f), lds(xaddr[q][2 * j + 1], 0.f));
    float u[D], zn[D];
#pragma unroll
    for (int j = 0; j < D / 2; ++j) {
      u2[j] = __fadd2_rn(__ffma2_rn(rho2, gx2[j], __fmul2_rn(omr2, zp[kF64 ? 0 : q][kF64 ? 0 : j])), lp[kF64 ? 0 : q][kF64 ? 0 : j]);
      u[2 * j] = u2[j].x;
      u[2 * j + 1] = u2[j].y;
    }
    project_pp_fixed<float, D>(u, zn);
    // idle checks run on the part's spare slot, whose x, z, l and messages stay
    // exactly 0 (u = 0 projects to 0): their residuals are 0, no predicate
#pragma unroll
    for (int j = 0; j < D / 2; ++j) {
      const float2 zn2 = make_float2(zn[2 * j], zn[2 * j + 1]);
      const float2 r1 = fsub2_rn(gx2[j], zn2);
      const float2 r2 = fsub2_rn(zn2, zp[kF64 ? 0 : q][kF64 ? 0 : j]);
      pr2 = __ffma2_rn(r1, r1, pr2);
      mv2 = __ffma2_rn(r2, r2, mv2);
      const float2 ln = fsub2_rn(u2[j], zn2);  // l' = (w + l) - z' = u - z'
      const float2 m2 = fsub2_rn(zn2, ln);
      lp[kF64 ? 0 : q][kF64 ? 0 : j] = ln;
      zp[kF64 ? 0 : q][kF64 ? 0 : j] = zn2;
      sts(xaddr[q][2 * j] + mstride * (1 + (2 * j) % DV), m2.x);
      sts(xaddr[q][2 * j + 1] + mstride * (1 + (2 * j + 1) % DV), m2.y);
    }
    }
  };

  // zero the whole local slot space once (ghost / spare slots hold finite values)
  for (int i = tid; i < NPL * (DV + 2); i += NT) sts(xs_a + ES * i, T(0));
  if (MBAR && tid == 0) {
    mbar_init(mb_x, 1);
    mbar_init(mb_m, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (PROF && tid == 0) {  // placement: which CTAs share an SM (tools/cluster_phases.py --placement)
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    printf("cta %d cluster %d rank %u smid %u\n", blockIdx.x, blockIdx.x / C, rank, smid);
  }
  uint32_t gi = 0;  // iterations run by this CTA (all frames): mbarrier phase parity
  __syncthreads();
  cl_barrier();  // every CTA of the cluster is running before any DSMEM access

  for (;;) {
    if (rank == 0 && tid == 0) {
      const int f = atomicAdd(p.queue, 1);
      for (uint32_t r = 0; r < C; ++r) cl_st_u32(cl_addr<C>(smem_u32(misc), r), static_cast<uint32_t>(f));
    }
    cl_barrier();
    const long long f = static_cast<int>(*reinterpret_cast<volatile int*>(misc));
    if (f >= p.batch) break;

    // ---- frame setup: gamma/mu of own variables, zero messages and state ----
#pragma unroll
    for (int q = 0; q < VPT; ++q) {
      const int v = vorig(q);
      const T g = v >= 0 ? div_rn(frame_llr<T>(p, f, v), p.mu) : T(0);  // fp32: __fdividef
      sts(xst(q) + mstride * (DV + 1), g);
#pragma unroll
      for (int j = 0; j < DV; ++j) sts(xst(q) + mstride * (j + 1), T(0));
    }
#pragma unroll
    for (int q = 0; q < CPT; ++q) {
      if constexpr (kF64) {
#pragma unroll
        for (int k = 0; k < D; ++k) {
          zd[q][k] = 0.0;
          ld[q][k] = 0.0;
        }
      } else {
#pragma unroll
        for (int j = 0; j < D / 2; ++j) {
          zp[kF64 ? 0 : q][kF64 ? 0 : j] = make_float2(0.f, 0.f);
          lp[kF64 ? 0 : q][kF64 ? 0 : j] = make_float2(0.f, 0.f);
        }
      }
    }
    if (tid == 0) {
      misc[1] = 0;
      if (!kF64) {  // fixed-point stop-rule accumulators, both parities
        sts4u(smem_u32(red), 0u);
        sts4u(smem_u32(red) + 16, 0u);
      }
    }
    __syncthreads();

    int t = 0;
    bool converged = false;
    if (prof) tp = clock64();
    for (;;) {
      ++t;
      if (prof) g_cl_cycles[7]++;
      phase(0);
      // ---- x-update of the own variables ----
#pragma unroll
      for (int h = 0; h < VPT / 2; ++h)
        var_pair(h);
      ADMM_JITTER();
      __syncthreads();
      // (fp32 stop-rule accumulators: the buffer of iteration gi + 1 was last
      // read in iteration gi - 1, which every thread left before this barrier)
      if (!kF64 && tid == 0) sts4u(smem_u32(red) + 16u * ((gi + 1) & 1), 0u);
      phase(1);
      // ---- x-send: own x -> ghost slots of the other CTAs (coalesced per warp) ----
      exchange(tx_b, p.n_xs[rank], mb_x);
      pr2 = make_float2(0.f, 0.f);
      mv2 = make_float2(0.f, 0.f);
      prd = mvd = 0.0;
      phase(2);
      ADMM_JITTER();
      if constexpr (MBAR) {
        if (tid == 0) mbar_expect(mb_x, p.rx_x[rank]);
        mbar_wait(mb_x, gi & 1);  // A: every ghost x of this iteration landed
      } else {
        cl_barrier();  // A: ghost x visible; every CTA done with its message rows
      }
      phase(3);
#pragma unroll
      for (int q = 0; q < CPT; ++q) check(q);

      const T primal = kF64 ? T(prd) : T(pr2.x + pr2.y), moved = kF64 ? T(mvd) : T(mv2.x + mv2.y);
      ADMM_JITTER();
      const int nc = __syncthreads_or(primal >= p.thr || moved >= p.thr);
      double sa = 0.0, sb = 0.0;
      if constexpr (!kF64) {
        // fp32: exact, order-free CTA sums in 42-bit fixed point (every partial
        // is below thr; resident_regular.cuh has the derivation): ~35
        // instructions where the fp64 butterfly costs ~125 -- on low-SNR points
        // the stuck frames take this path in most iterations.  The header
        // carries the 64-bit integers in its double slots.
        if (!nc) {
          uint32_t* fx = reinterpret_cast<uint32_t*>(red) + 4 * (gi & 1);
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
          const uint4 v = lds4u(smem_u32(fx));
          sa = __longlong_as_double(static_cast<long long>((static_cast<unsigned long long>(v.x) << 21) + v.y));
          sb = __longlong_as_double(static_cast<long long>((static_cast<unsigned long long>(v.z) << 21) + v.w));
        }
      } else if (!nc) {  // fp64: exact CTA sums in fp64 (fixed order)
        const double wa = warp_allsum(static_cast<double>(primal));
        const double wb = warp_allsum(static_cast<double>(moved));
        if (lane == 0) {
          red[2 * warp] = wa;
          red[2 * warp + 1] = wb;
        }
        __syncthreads();
        const double a = lane < nwarps ? red[2 * lane] : 0.0;
        const double b = lane < nwarps ? red[2 * lane + 1] : 0.0;
        sa = warp_allsum(a);
        sb = warp_allsum(b);
      }
      phase(4);
      // ---- msg-send: ghost-row messages -> the owners' message rows; stop-rule header ----
      exchange(tm_b, p.n_ms[rank], mb_m);
      if (tid < C) {
        const uint32_t r = tid;
        ClusterHeader* h = hdr + (MBAR ? (gi & 1) : 0);
        if constexpr (MBAR) {
          const uint32_t mb = cl_addr<C>(mb_m, r, 8);
          cl_st_async_f64(cl_addr<C>(smem_u32(&h->primal[rank]), r, 8), sa, mb);
          cl_st_async_f64(cl_addr<C>(smem_u32(&h->moved[rank]), r, 8), sb, mb);
          cl_st_async_u32(cl_addr<C>(smem_u32(&h->flag[rank]), r), static_cast<uint32_t>(nc), mb);
        } else {
          cl_st_f64(cl_addr<C>(smem_u32(&h->primal[rank]), r, 8), sa);
          cl_st_f64(cl_addr<C>(smem_u32(&h->moved[rank]), r, 8), sb);
          cl_st_u32(cl_addr<C>(smem_u32(&h->flag[rank]), r), static_cast<uint32_t>(nc));
        }
      }
      phase(5);
      ADMM_JITTER();
      if constexpr (MBAR) {
        if (tid == 0) mbar_expect(mb_m, p.rx_m[rank]);
        mbar_wait(mb_m, gi & 1);  // B: our messages and every CTA's header landed
      } else {
        cl_barrier();  // B: messages and headers visible
      }
      const ClusterHeader* hd = hdr + (MBAR ? (gi & 1) : 0);
      ++gi;
      // flags first; the fp64 sums only when every CTA's partials were below
      // the threshold (rare)
      uint32_t anync = 0;
#pragma unroll
      for (int r = 0; r < C; r += 4) {
        const uint4 fl = lds4u(smem_u32(&hd->flag[r]));  // C is 4 or 8
        anync |= fl.x | fl.y | fl.z | fl.w;
      }
      phase(6);
      if (!anync) {
        bool conv;
        if constexpr (kF64) {
          double A = 0.0, B = 0.0;
#pragma unroll
          for (int r = 0; r < C; ++r) {
            A += hd->primal[r];
            B += hd->moved[r];
          }
          conv = A < p.thr_d && B < p.thr_d;
        } else {
          unsigned long long A = 0, B = 0;
#pragma unroll
          for (int r = 0; r < C; ++r) {
            A += static_cast<unsigned long long>(__double_as_longlong(hd->primal[r]));
            B += static_cast<unsigned long long>(__double_as_longlong(hd->moved[r]));
          }
          conv = A < p.fx_thr && B < p.fx_thr;
        }
        if (conv) {
          converged = true;
          break;
        }
      }
      if (t >= p.t_max) break;
    }

    // ---- outputs (make_output, admm_decoder.py:92-105; is_codeword, codes.py:145-154) ----
    bool integral = true;
    int ones = 0;
#pragma unroll
    for (int q = 0; q < VPT; ++q) {
      const int v = vorig(q);
      if (v >= 0) {
        const T xv = lds(xst(q), T());
        const bool h = xv > T(0.5);
        ones += h;
        integral &= vmin(fabs(xv), fabs(T(1) - xv)) <= T(1e-5);
        ADMM_ASSERT(v < p.n_vars && f < p.batch);
        if (p.x_out) p.x_out[f * p.ld_x + v] = xv;
        if (p.hard_out) p.hard_out[f * p.ld_hard + v] = h;
      }
    }
    bool odd = false;
#pragma unroll
    for (int q = 0; q < CPT; ++q) {
      int par = 0;
#pragma unroll
      for (int k = 0; k < D; ++k) par ^= (lds(xaddr[q][k], T()) > T(0.5));
      odd |= ((cmask >> q) & 1u) && par;
    }
    ones = __reduce_add_sync(0xffffffffu, ones);
    if (lane == 0 && ones) atomicAdd(misc + 1, ones);
    const int all_integral = __syncthreads_and(integral);
    const int any_odd = __syncthreads_or(odd);
    if (tid == 0) {
      const uint32_t o = cl_addr<C>(smem_u32(outslot + 3 * rank), 0, 4);
      cl_st_u32(o, static_cast<uint32_t>(all_integral));
      cl_st_u32(o + 4, static_cast<uint32_t>(misc[1]));
      cl_st_u32(o + 8, static_cast<uint32_t>(any_odd));
    }
    cl_barrier();
    if (rank == 0 && tid == 0) {
      int integ = 1, wt = 0, oddc = 0;
      for (int r = 0; r < C; ++r) {
        integ &= outslot[3 * r] != 0;
        wt += outslot[3 * r + 1];
        oddc |= outslot[3 * r + 2];
      }
      if (p.iters_out) p.iters_out[f] = t;
      if (p.flags_out)
        p.flags_out[f] = (converged ? kFlagConverged : 0) | (integ ? kFlagIntegral : 0) | (oddc ? 0 : kFlagCodeword);
      if (p.weight_out) p.weight_out[f] = wt;
    }
  }
}

}  // namespace admm
