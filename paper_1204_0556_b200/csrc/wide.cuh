// Wide streaming engine: large batches of frames of codes that do not fit one
// SM (BASELINE config 5, n = 16384), with the decoder state in HBM.
//
// The sharded engine (sharded.cuh) keeps z/lambda in shared memory and can
// therefore hold only ~64 frame slots; its passes are short (~25 us) and
// bound by L2 latency and grid syncs.  This engine instead streams the whole
// state through HBM every pass over S = 1024-8192 slots, so each phase is a
// long, fully parallel, bandwidth-bound sweep -- the two-kernel HBM schedule
// of SURVEY.md 8d (28 B per edge-update in fp32):
//
//   phase V (variables)  read messages (DV per variable) + gamma/mu, write x
//                        (admm_decoder.py:108-124)
//   phase C (checks)     gather x, read the edge state, fused z-update,
//                        projection, residual partials, lambda-update; write
//                        the edge state and the messages z - lambda/mu
//                        (admm_decoder.py:127-149, parity_polytope.py:352-421)
//   phase S (slots)      exact stop rule (:169, 174-181), retirement, refill
//
// Layout: slots are grouped in STRIPES of W = 32*VS consecutive slots (VS = 2
// fp32 / 1 fp64 slots per lane); every array is stripe-major, then row (edge
// or variable), then the stripe's 32 lanes x VS slots:
//     zl  [stripe][E][32][VS] z (fp32; the messages hold z - lambda/mu)
//         [stripe][E][32][2][VS] z and lambda/mu (fp64)
//     msg [stripe][E][32][VS]   x, gm [stripe][N][32][VS]
//     part[stripe][ncb][2][32][VS] per-check-block residual partials
// so a warp's access to one row is one contiguous 256-byte segment (512 for
// the fp64 edge state); the rows of the checks of one work item are
// contiguous.
//
// Work items are (stripe, block of rows), taken dynamically by warps in
// stripe-major order (ItemFeed below), moved through a per-warp cp.async
// ring of shared-memory stages.  No __syncthreads in the phases; phases are
// separated by grid syncs of the cooperative kernel.
//
// Slot life: FRESH (z = lambda = 0 implicit) -> RUNNING -> next frame, or
// EMPTY.  Phase V accumulates the output statistics of every new x and phase
// C the syndrome of its hard decision, so phase S retires a converged frame
// in the pass that converged it; only when x or hard decisions are requested
// does the slot spend a RETIRING pass writing them.  The stop rule is exact:
// the S phase sums the per-block partials of every running slot in a fixed
// order (lane-strided blocks + butterfly), so decisions are deterministic and
// independent of the batch composition.
#pragma once

#include <cooperative_groups.h>

#include "common.cuh"
#include "projection.cuh"
#include "streaming.cuh"
#include "synth.cuh"

namespace admm {

template <typename T, int VS>
struct alignas(sizeof(T) * VS) WVec {
  T v[VS];
};

constexpr int kWideThreads = 256;
constexpr int kWideCB = 8;   // checks per phase-C work item (one warp)
constexpr int kWideVB = 16;  // variables per phase-V work item (one warp)

template <typename T>
struct WideParams {
  int n_vars, n_checks, n_edges, m_pad, dvmax;
  const int* chk_var;    // [D][m_pad], -1 = unused
  const int* edge_base;  // [n_checks]
  const int* var_edge;   // [n_vars][dvmax], -1 = unused
  const int* ctbl;       // [ncb][wide_ct(D)] check-block index tables
  const int* vtbl;       // [nvb][wide_vt(DVMAX)] variable-block index tables
  long long batch;
  const T* gamma;
  long long ld_gamma;
  T mu, rho, one_minus_rho, thr;  // thr: eps^2 E rounded up to T (early-out tests)
  double thr_d;                    // eps^2 E: the exact sums are fp64
  int t_max;
  T* x_out;
  long long ld_x;
  uint8_t* hard_out;
  long long ld_hard;
  int* iters_out;
  uint8_t* flags_out;
  int* weight_out;
  int S, ncb;
  T* zl;
  T* msg;
  T* x;
  T* gm;
  T* part;
  T* gfr;    // [S][N] LLRs of the slots' next frames (in-kernel synthesis only)
  int* vpart;  // [stripe][nvb][W] hard-decision weight | non-integral << 8 of x per variable block (every pass)
  int direct;  // no per-variable outputs requested: retire without the retiring pass
  int* frame;  // [S] frame of the slot
  int* fnext;  // [S] frame that follows a retiring slot's frame (-1 = none)
  int* slist;  // [S] slots whose next frame's LLRs are synthesised in the coming pass
  int *st, *tcount, *conv, *weight, *nonint, *odd, *ctr;
  SynthParams synth;
};

struct WideLayout {
  size_t zl, msg, x, gm, part, gfr, vpart, ints, total;
  static size_t al(size_t b) { return (b + 255) & ~size_t(255); }
  WideLayout(size_t elem, long long E, long long N, long long ncb, long long S, bool synth) {
    size_t o = 0;
    zl = o; o += al(elem * (elem == 4 ? 1 : 2) * E * S);  // fp32: z only (the message array holds z - lambda/mu)
    msg = o; o += al(elem * E * S);
    x = o; o += al(elem * N * S);
    gm = o; o += al(elem * N * S);
    part = o; o += al(elem * 2 * ncb * S);
    gfr = o; o += synth ? al(elem * N * S) : 0;
    vpart = o; o += al(sizeof(int) * ((N + kWideVB - 1) / kWideVB) * S);
    ints = o; o += al(sizeof(int) * (10 * S + 16));
    total = o;
  }
};

template <typename V>
__device__ __forceinline__ V wld(const V* p) { return *p; }
template <typename V>
__device__ __forceinline__ void wst(V* p, const V& v) { *p = v; }

// Streaming stores (st.global.cs: evict-first) for the state written once
// per pass and read back only in the next one: edge state, messages, gamma/mu.
template <typename V>
__device__ __forceinline__ void st_cs(V* p, const V& v) {
  if constexpr (sizeof(V) == 32) {
    float4 t0, t1;
    memcpy(&t0, &v, 16);
    memcpy(&t1, reinterpret_cast<const char*>(&v) + 16, 16);
    __stcs(reinterpret_cast<float4*>(p), t0);
    __stcs(reinterpret_cast<float4*>(p) + 1, t1);
  } else if constexpr (sizeof(V) == 16) {
    float4 t;
    memcpy(&t, &v, 16);
    __stcs(reinterpret_cast<float4*>(p), t);
  } else if constexpr (sizeof(V) == 8) {
    float2 t;
    memcpy(&t, &v, 8);
    __stcs(reinterpret_cast<float2*>(p), t);
  } else {
    float t;
    memcpy(&t, &v, 4);
    __stcs(reinterpret_cast<float*>(p), t);
  }
}

// ---- per-warp cp.async pipeline ----
// Every lane copies its own vectors into its warp's ring of NS stages and
// reads back only what it copied, so a stage needs no barrier: wait_group
// makes a lane's copies visible to it.  The loads of task t+NS-1 are in
// flight while task t computes, and the in-flight bytes live in shared
// memory instead of registers.
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}
template <int BYTES>
__device__ __forceinline__ void cp_async_vec(uint32_t dst, const void* src) {
  if constexpr (BYTES == 32) {
    cp_async16(dst, src);
    cp_async16(dst + 16, static_cast<const char*>(src) + 16);
  } else if constexpr (BYTES == 16) {
    cp_async16(dst, src);
  } else if constexpr (BYTES == 8) {
    cp_async8(dst, src);
  } else {
    static_assert(BYTES == 4, "vector size");
    cp_async4(dst, src);
  }
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
template <typename V>
__device__ __forceinline__ V lds_vec(const unsigned char* p) {
  return *reinterpret_cast<const V*>(p);
}

// Stage geometry.  A stage holds one task: for a check task D x-rows and D
// edge-state rows, for a variable task VBB variables x (DVMAX message rows,
// gamma/mu, x, fresh LLR) -- each row 32 lanes x one vector.
template <typename T, int VS, int D, int DVMAX>
struct WideStage {
  static constexpr int VB = VS * static_cast<int>(sizeof(T));  // bytes per lane per row
  static constexpr int CX = 0, CZ = D * 32 * VB;                 // check task: x rows, edge-state rows
  static constexpr int CBYTES = D * 32 * 3 * VB;
  static constexpr int VROWS = DVMAX + 3;                        // messages, gamma/mu, x, fresh LLRs
  static constexpr int VBB = (3 * D) / VROWS > 0 ? (3 * D) / VROWS : 1;
  static constexpr int VBYTES = VBB * VROWS * 32 * VB;
  static constexpr int bytes = ((CBYTES > VBYTES ? CBYTES : VBYTES) + 15) / 16 * 16;
};

// ---- work items ----
// The stripes form two groups, G0 and G1, half a pass out of phase: one
// STEP runs the variable phase of one group together with the check phase of
// the other, so the latency-bound variable work (random message-row gathers)
// and the bandwidth-bound check work share the SMs and HBM instead of
// alternating; a pass is two steps, each followed by the slot phase of the
// group whose check phase just finished.
//
// Within a step, items are (stripe, block of kWideVB variables) of the V
// group and (stripe, block of kWideCB checks) of the C group, numbered
// stripe-major and interleaved V, C, V, C, ...  Warps take them dynamically
// from a global counter (a static split left a quarter of the SM time
// waiting at the grid syncs).  For the item after the current one the feed
// prefetches (into registers) the block's precomputed index table (wide_ct /
// wide_vt ints, one coalesced access per lane) and the lane's slot states and
// frames, and publishes them to the warp's shared-memory table slot when the
// item starts: no copy issue and no compute step ever waits on a dependent
// index or state load.
__host__ __device__ constexpr int wide_ct(int D) { return ((D + 1) * kWideCB + 31) / 32 * 32; }
__host__ __device__ constexpr int wide_vt(int DV) { return (kWideVB * DV + 31) / 32 * 32; }
template <int D, int DVMAX>
__host__ __device__ constexpr int wide_tbmax() {
  return wide_ct(D) > wide_vt(DVMAX) ? wide_ct(D) : wide_vt(DVMAX);
}
// Table slot: [TBM index ints][id, stripe, block, busy, kind, -, -, -][32 x VS states][32 x VS frames]
template <int D, int DVMAX, int VS>
__host__ __device__ constexpr int wide_tstride() {
  return wide_tbmax<D, DVMAX>() + 8 + 64 * VS;
}
enum : int { kItemV = 0, kItemC = 1 };

// The items of one step: nv variable items of stripes [vs0, vs0 + nvs) and
// nc check items of stripes [cs0, cs0 + ncs).
struct WideStep {
  int vs0, nvs, cs0, ncs;
  int n_vb, ncb;
  int nv, nc, m, total;
  __device__ __forceinline__ WideStep(int vs0_, int nvs_, int cs0_, int ncs_, int n_vb_, int ncb_)
      : vs0(vs0_), nvs(nvs_), cs0(cs0_), ncs(ncs_), n_vb(n_vb_), ncb(ncb_) {
    nv = nvs * n_vb;
    nc = ncs * ncb;
    m = nv < nc ? nv : nc;
    total = nv + nc;
  }
  // item k -> kind, stripe, block
  __device__ __forceinline__ void decode(int k, int& kind, int& stripe, int& block) const {
    int idx;
    if (k < 2 * m) {
      kind = k & 1;
      idx = k >> 1;
    } else {
      kind = nv > nc ? kItemV : kItemC;
      idx = k - m;
    }
    if (kind == kItemV) {
      stripe = vs0 + idx / n_vb;
      block = idx % n_vb;
    } else {
      stripe = cs0 + idx / ncb;
      block = idx % ncb;
    }
  }
};

template <int TBV, int TBC, int VS>
struct ItemFeed {
  static constexpr int TBM = TBV > TBC ? TBV : TBC;
  static constexpr int NR = TBM / 32;
  using VI = WVec<int, VS>;
  const int* vtbl;  // [n_vb][TBV]
  const int* ctbl;  // [ncb][TBC]
  int* ctr;
  const WideStep* stp;
  int W;
  const int* st;
  const int* frame;
  int id1;         // next item (its table/states are in registers)
  int raw2, raw3;  // lane 0: atomic results for the two items after (in flight)
  int kind1, stripe1, block1;
  int reg[NR];
  VI sreg, freg;

  __device__ __forceinline__ int grab_raw() { return (threadIdx.x & 31) == 0 ? atomicAdd(ctr, 1) : 0; }
  __device__ __forceinline__ void load(int id) {
    if (id < stp->total) {
      const int lane = threadIdx.x & 31;
      stp->decode(id, kind1, stripe1, block1);
      const int tb = kind1 == kItemV ? TBV : TBC;
      const int* t = (kind1 == kItemV ? vtbl : ctbl) + (long long)block1 * tb + lane;
#pragma unroll
      for (int r = 0; r < NR; ++r)
        if (r * 32 < tb) reg[r] = __ldg(t + r * 32);
      const int s0 = stripe1 * W + lane * VS;
      sreg = *reinterpret_cast<const VI*>(st + s0);
      freg = *reinterpret_cast<const VI*>(frame + s0);
    }
  }
  __device__ __forceinline__ void publish(int* slot, int id) {
    const int lane = threadIdx.x & 31;
    __syncwarp();  // every lane is done reading the slot's previous contents
#pragma unroll
    for (int r = 0; r < NR; ++r) slot[r * 32 + lane] = reg[r];
    bool act = false;
#pragma unroll
    for (int l = 0; l < VS; ++l) act |= sreg.v[l] != kSlotEmpty;
    act = __any_sync(0xffffffffu, act);
    if (lane == 0) {
      slot[TBM] = id;
      slot[TBM + 1] = stripe1;
      slot[TBM + 2] = block1;
      slot[TBM + 3] = act;  // any slot of the item's stripe lanes busy
      slot[TBM + 4] = kind1;
    }
    *reinterpret_cast<VI*>(slot + TBM + 8 + lane * VS) = sreg;
    *reinterpret_cast<VI*>(slot + TBM + 8 + 32 * VS + lane * VS) = freg;
    __syncwarp();
  }
  // First item: published into slot0; returns its id.
  __device__ __forceinline__ int start(int* slot0) {
    const int a = __shfl_sync(0xffffffffu, grab_raw(), 0);
    id1 = __shfl_sync(0xffffffffu, grab_raw(), 0);
    load(a);
    publish(slot0, a);
    load(id1);
    raw2 = grab_raw();
    raw3 = grab_raw();
    return a;
  }
  // Move to the next item: publish it into `slot`, prefetch the one after.
  __device__ __forceinline__ int advance(int* slot) {
    const int cur = id1;
    publish(slot, cur);
    id1 = __shfl_sync(0xffffffffu, raw2, 0);
    load(id1);
    raw2 = raw3;
    raw3 = grab_raw();
    return cur;
  }
};

// Shared memory: per warp two table slots and the ring of NS stages.
template <typename T, int VS, int D, int DVMAX, int NS>
__host__ __device__ constexpr int wide_warp_bytes() {
  return 2 * 4 * wide_tstride<D, DVMAX, VS>() + NS * WideStage<T, VS, D, DVMAX>::bytes;
}
template <typename T, int VS, int D, int DVMAX, int NS>
__host__ __device__ constexpr int wide_smem_bytes() {
  return (kWideThreads / 32) * wide_warp_bytes<T, VS, D, DVMAX, NS>();
}

// LLRs of the next frames of slots that started a frame in the last slot
// phase (in-kernel synthesis): written slot-major, one lane per variable,
// while the current frame runs, so the first x-update of the next frame
// reads them like a stored LLR vector instead of running Philox +
// Box-Muller on a few lanes of every warp.
constexpr int kWideSynthChunk = 2048;

template <typename T>
__device__ __forceinline__ void wide_synth_items(const WideParams<T>& p, const int* list, int nlist, int* grab) {
  const int lane = threadIdx.x & 31;
  const int nch = (p.n_vars + kWideSynthChunk - 1) / kWideSynthChunk;
  const int n = nlist * nch;
  for (;;) {
    const int q = __shfl_sync(0xffffffffu, lane == 0 ? atomicAdd(grab, 1) : 0, 0);
    if (q >= n) break;
    const int s = list[q / nch], c = q % nch;
    const int f = p.fnext[s];
    const int i1 = min(p.n_vars, (c + 1) * kWideSynthChunk);
    for (int i = c * kWideSynthChunk + lane; i < i1; i += 32)
      p.gfr[(long long)s * p.n_vars + i] = static_cast<T>(synth_llr(p.synth, p.synth.trial0 + f, i));
  }
}

// Edge-state store of phase C: (z, lambda/mu) pairs, or z alone (ZM).
template <typename T, int VS, bool ZM>
__device__ __forceinline__ void wide_store_z(WVec<T, 2 * VS>* zl, WVec<T, VS>* zv, long long row,
                                             const WVec<T, 2 * VS>& v) {
  if constexpr (ZM) {
    WVec<T, VS> z;
#pragma unroll
    for (int l = 0; l < VS; ++l) z.v[l] = v.v[l];
    wst(zv + row, z);
  } else {
    wst(zl + row, v);
  }
}

// ---- one step: phase V of one stripe group, phase C of the other ----
//
// phase V: x = clip((sum msg - gamma/mu) / deg) (admm_decoder.py:108-124).
// One code path for every slot state (per-lane selects): a FRESH slot sums no
// messages and takes gamma/mu from its frame's LLR vector; a RETIRING slot
// keeps x and accumulates the output statistics (make_output, :92-105).
//
// phase C: fused z-update, projection, residuals, lambda-update, message
// (admm_decoder.py:127-149, parity_polytope.py:352-421).  FRESH slots start
// from z = lambda = 0, only RUNNING/FRESH slots add to the residual partials,
// every slot adds the parity of its hard decision (is_codeword,
// codes.py:145-154) to the block's syndrome flag.
template <typename T, int VS, int D, int DVMAX, bool REG, int NS>
__device__ __forceinline__ void wide_step(const WideParams<T>& p, unsigned char* ring, int* tslot, int tstride,
                                          const WideStep& sp, int* ctr_items) {
  using V = WVec<T, VS>;
  using VI = WVec<int, VS>;
  using V2 = WVec<T, 2 * VS>;
  using G = WideStage<T, VS, D, DVMAX>;
  constexpr int W = 32 * VS, VBB = G::VBB, VB = G::VB, CB = kWideCB;
  constexpr int TPIV = (kWideVB + VBB - 1) / VBB;
  constexpr int TBV = wide_vt(DVMAX), TBC = wide_ct(D), TBM = wide_tbmax<D, DVMAX>();
  constexpr int ES = static_cast<int>(sizeof(T));
  // fp32 keeps (z, message) per edge and recovers lambda/mu = z - message:
  // 20 instead of 24 bytes of edge-state traffic per edge-update.  fp64 (the
  // parity mode) keeps (z, lambda/mu) and writes the message separately.
  constexpr bool ZM = sizeof(T) == 4;
  static_assert(NS - 1 < TPIV && NS - 1 < CB, "stage ring deeper than an item");
  const int lane = threadIdx.x & 31;
  const long long E = p.n_edges, N = p.n_vars;
  V* x = reinterpret_cast<V*>(p.x);
  V* gm = reinterpret_cast<V*>(p.gm);
  V2* zl = reinterpret_cast<V2*>(p.zl);
  V* zv = reinterpret_cast<V*>(p.zl);
  V* msg = reinterpret_cast<V*>(p.msg);
  const int n_vb = sp.n_vb, ncb = sp.ncb, n_items = sp.total;
  const uint32_t ring_s = smem_u32(ring);
  ItemFeed<TBV, TBC, VS> feed{p.vtbl, p.ctbl, ctr_items, &sp, W, p.st, p.frame};
  int ik = 0, iq = 0, ti = 0;
  int iid = feed.start(tslot);

  auto issue_next = [&]() {
    __syncwarp();
    const int* tb = tslot + (ik & 1) * tstride;
    const int kind = tb[TBM + 4];
    if (iid < n_items) {
      const int stripe = tb[TBM + 1], blk = tb[TBM + 2];
      const uint32_t st = ring_s + (ti % NS) * G::bytes;
      if (kind == kItemV) {
        const int i0 = blk * kWideVB + iq * VBB, i1 = min(p.n_vars, min((blk + 1) * kWideVB, i0 + VBB));
        if (tb[TBM + 3] && i0 < i1) {
          const VI stv = *reinterpret_cast<const VI*>(tb + TBM + 8 + lane * VS);
          const VI frv = *reinterpret_cast<const VI*>(tb + TBM + 8 + 32 * VS + lane * VS);
          bool anyret = false;
#pragma unroll
          for (int l = 0; l < VS; ++l) anyret |= stv.v[l] == kSlotRetiring;
          const long long rb = (long long)stripe * N * 32 + lane;
#pragma unroll
          for (int b = 0; b < VBB; ++b) {
            const int i = i0 + b;
            if (i < i1) {
              const uint32_t rowb = st + b * G::VROWS * 32 * VB + lane * VB;
#pragma unroll
              for (int j = 0; j < DVMAX; ++j) {
                const int e = tb[(iq * VBB + b) * DVMAX + j];
                if (e >= 0) cp_async_vec<VB>(rowb + j * 32 * VB, msg + ((long long)stripe * E + e) * 32 + lane);
              }
              cp_async_vec<VB>(rowb + DVMAX * 32 * VB, gm + rb + (long long)i * 32);
              if (anyret) cp_async_vec<VB>(rowb + (DVMAX + 1) * 32 * VB, x + rb + (long long)i * 32);
#pragma unroll
              for (int l = 0; l < VS; ++l) {
                if (stv.v[l] != kSlotFresh) continue;
                const T* src = p.synth.kind != 0 ? p.gfr + (long long)(stripe * W + lane * VS + l) * N + i
                                                 : p.gamma + (long long)frv.v[l] * p.ld_gamma + i;
                cp_async_vec<ES>(rowb + (DVMAX + 2) * 32 * VB + l * ES, src);
              }
            }
          }
        }
      } else {
        const int c = blk * CB + iq;
        if (tb[TBM + 3] && c < p.n_checks) {
          const long long e0 = tb[D * CB + iq];
          const long long xb = (long long)stripe * N * 32 + lane, eb = (long long)stripe * E * 32 + lane;
#pragma unroll
          for (int k = 0; k < D; ++k) {
            const int v = tb[k * CB + iq];
            if (v >= 0) {
              cp_async_vec<VB>(st + G::CX + (k * 32 + lane) * VB, x + xb + (long long)v * 32);
              if constexpr (ZM) {
                cp_async_vec<VB>(st + G::CZ + (k * 32 + lane) * 2 * VB, zv + eb + (e0 + k) * 32);
                cp_async_vec<VB>(st + G::CZ + (k * 32 + lane) * 2 * VB + VB, msg + eb + (e0 + k) * 32);
              } else {
                cp_async_vec<2 * VB>(st + G::CZ + (k * 32 + lane) * 2 * VB, zl + eb + (e0 + k) * 32);
              }
            }
          }
        }
      }
    }
    cp_commit();
    ++ti;
    if (++iq == (kind == kItemV ? TPIV : CB)) {
      iq = 0;
      ++ik;
      iid = feed.advance(tslot + (ik & 1) * tstride);
    }
  };

  // per-item accumulators (phase V: weight / non-integral of the new x;
  // phase C: residual partials and the syndrome flag), flushed at item ends
  int iw[VS], inon[VS], odd[VS];
  T primal[VS], moved[VS];
#pragma unroll
  for (int l = 0; l < VS; ++l) {
    iw[l] = inon[l] = odd[l] = 0;
    primal[l] = moved[l] = T(0);
  }
#pragma unroll
  for (int t = 0; t < NS - 1; ++t) issue_next();
  int ck = 0, cq = 0;
  for (int t = 0;; ++t) {
    const int* tb = tslot + (ck & 1) * tstride;
    const int cid = tb[TBM];
    if (cid >= n_items) break;
    const int kind = tb[TBM + 4];
    const int cqt = cq;
    if (++cq == (kind == kItemV ? TPIV : CB)) {
      cq = 0;
      ++ck;
    }
    issue_next();
    cp_wait<NS - 1>();
    const int stripe = tb[TBM + 1], blk = tb[TBM + 2];
    if (!tb[TBM + 3]) continue;  // every slot of the stripe empty
    const unsigned char* st = ring + (t % NS) * G::bytes;
    const VI stv = *reinterpret_cast<const VI*>(tb + TBM + 8 + lane * VS);
    const int s0 = stripe * W + lane * VS;
    if (kind == kItemV) {
      // ---------------- phase V task: VBB variables ----------------
      const int i0 = blk * kWideVB + cqt * VBB, i1 = min(p.n_vars, min((blk + 1) * kWideVB, i0 + VBB));
      if (i0 >= i1) continue;
      const VI frv = *reinterpret_cast<const VI*>(tb + TBM + 8 + 32 * VS + lane * VS);
      bool anyupd = false, anyfresh = false, anyret = false;
#pragma unroll
      for (int l = 0; l < VS; ++l) {
        anyupd |= stv.v[l] != kSlotEmpty;
        anyfresh |= stv.v[l] == kSlotFresh;
        anyret |= stv.v[l] == kSlotRetiring;
      }
      int wsum[VS], nonint[VS];
#pragma unroll
      for (int l = 0; l < VS; ++l) wsum[l] = nonint[l] = 0;
      const long long rb = (long long)stripe * N * 32 + lane;
#pragma unroll
      for (int b = 0; b < VBB; ++b) {
        const int i = i0 + b;
        if (i >= i1) break;
        const unsigned char* rowb = st + b * G::VROWS * 32 * VB + lane * VB;
        int deg = 0;
        V mv[DVMAX];
#pragma unroll
        for (int j = 0; j < DVMAX; ++j) {
          const bool on = REG || tb[(cqt * VBB + b) * DVMAX + j] >= 0;
          deg += on;
          if (on) mv[j] = lds_vec<V>(rowb + j * 32 * VB);
        }
        V g = lds_vec<V>(rowb + DVMAX * 32 * VB);
        V xo, gf;
        if (anyret) xo = lds_vec<V>(rowb + (DVMAX + 1) * 32 * VB);
        if (anyfresh) gf = lds_vec<V>(rowb + (DVMAX + 2) * 32 * VB);
        V xn;
#pragma unroll
        for (int l = 0; l < VS; ++l) {
          const int state = stv.v[l];
          const bool fresh = state == kSlotFresh, ret = state == kSlotRetiring;
          T acc = T(0);
#pragma unroll
          for (int j = 0; j < DVMAX; ++j)
            if (j < deg) acc = add_rn(acc, mv[j].v[l]);  // increasing edge id (np.bincount order)
          if (anyfresh) {
            if (fresh) acc = T(0);  // z = lambda = 0 (AdmmState.initial)
            g.v[l] = fresh ? div_rn(gf.v[l], p.mu) : g.v[l];
          }
          T xv = deg > 0 ? clip01(div_rn(sub_rn(acc, g.v[l]), T(deg))) : (g.v[l] < T(0) ? T(1) : T(0));
          iw[l] += xv > T(0.5) ? 1 : 0;  // make_output (:92-105) of x_t, in case the slot stops now
          inon[l] |= !(vmin(fabs(xv), fabs(T(1) - xv)) <= T(1e-5)) ? 1 : 0;
          if (anyret) {
            const T xf = xo.v[l];  // final iterate of a retiring slot
            const bool h = xf > T(0.5);
            wsum[l] += (ret && h) ? 1 : 0;
            nonint[l] |= (ret && !(vmin(fabs(xf), fabs(T(1) - xf)) <= T(1e-5))) ? 1 : 0;
            if (ret) {
              if (p.x_out) p.x_out[(long long)frv.v[l] * p.ld_x + i] = xf;
              if (p.hard_out) p.hard_out[(long long)frv.v[l] * p.ld_hard + i] = h;
              xv = xf;
            }
          }
          xn.v[l] = xv;
        }
        if (anyupd) wst(x + rb + (long long)i * 32, xn);
        if (anyfresh) st_cs(gm + rb + (long long)i * 32, g);
      }
      if (anyret) {
#pragma unroll
        for (int l = 0; l < VS; ++l) {
          if (wsum[l]) atomicAdd(p.weight + s0 + l, wsum[l]);
          if (nonint[l]) atomicOr(p.nonint + s0 + l, 1);
        }
      }
      if (i1 == min(p.n_vars, (blk + 1) * kWideVB)) {  // last task of the item
        if (p.direct) {
          VI o;
#pragma unroll
          for (int l = 0; l < VS; ++l) o.v[l] = iw[l] | (inon[l] << 8);
          *reinterpret_cast<VI*>(p.vpart + ((long long)stripe * n_vb + blk) * W + lane * VS) = o;
        }
#pragma unroll
        for (int l = 0; l < VS; ++l) iw[l] = inon[l] = 0;
      }
    } else {
      // ---------------- phase C task: one check ----------------
      const int c = blk * CB + cqt;
      if (c >= p.n_checks) continue;
      bool anyret = false;
#pragma unroll
      for (int l = 0; l < VS; ++l) anyret |= stv.v[l] == kSlotRetiring;
      int d = REG ? D : 0;
      if constexpr (!REG) {
#pragma unroll
        for (int k = 0; k < D; ++k) d += tb[k * CB + cqt] >= 0;
      }
      const long long e0 = tb[D * CB + cqt];
      const long long eb = (long long)stripe * E * 32 + lane;
      V gx[D];
      V2 zlv[D];
#pragma unroll
      for (int k = 0; k < D; ++k)
        if (k < d) {
          gx[k] = lds_vec<V>(st + G::CX + (k * 32 + lane) * VB);
          zlv[k] = lds_vec<V2>(st + G::CZ + (k * 32 + lane) * 2 * VB);
          if constexpr (ZM) {
#pragma unroll
            for (int l = 0; l < VS; ++l) zlv[k].v[VS + l] = sub_rn(zlv[k].v[l], zlv[k].v[VS + l]);
          }
        }
#pragma unroll
      for (int l = 0; l < VS; ++l) {
        int par = 0;
#pragma unroll
        for (int k = 0; k < D; ++k)
          if (k < d) par ^= gx[k].v[l] > T(0.5);
        odd[l] |= par;
      }
#pragma unroll
      for (int l = 0; l < VS; ++l) {
        const bool run = stv.v[l] == kSlotRunning;
        const bool act = run || stv.v[l] == kSlotFresh;
        T w_[D], u[D], zn[D], zo[D], lo[D];
#pragma unroll
        for (int k = 0; k < D; ++k) {
          const bool on = k < d;
          zo[k] = run ? zlv[k].v[l] : T(0);
          lo[k] = run ? zlv[k].v[VS + l] : T(0);  // scaled dual lambda/mu
          const T g = on ? gx[k].v[l] : T(0);
          w_[k] = add_rn(mul_rn(p.rho, g), mul_rn(p.one_minus_rho, zo[k]));
          u[k] = on ? add_rn(w_[k], lo[k]) : -Num<T>::inf();
        }
        if constexpr (REG) {
          project_pp_fixed<T, D>(u, zn);
        } else {
          project_pp<T, D>(u, zn, d);
        }
        T pr = T(0), mo = T(0);
#pragma unroll
        for (int k = 0; k < D; ++k) {
          if (k < d) {
            const T r1 = sub_rn(gx[k].v[l], zn[k]);
            const T r2 = sub_rn(zn[k], zo[k]);
            pr = add_rn(pr, mul_rn(r1, r1));
            mo = add_rn(mo, mul_rn(r2, r2));
            // fp32 (throughput mode): l' = (w + l) - z' = u - z' as in the
            // resident kernels; fp64 keeps the reference's expression tree
            const T lnew = ZM ? sub_rn(u[k], zn[k]) : add_rn(lo[k], sub_rn(w_[k], zn[k]));
            zlv[k].v[l] = zn[k];
            zlv[k].v[VS + l] = lnew;
            gx[k].v[l] = sub_rn(zn[k], lnew);  // message
          }
        }
        primal[l] = act ? add_rn(primal[l], pr) : primal[l];
        moved[l] = act ? add_rn(moved[l], mo) : moved[l];
      }
#pragma unroll
      for (int k = 0; k < D; ++k)
        if (k < d) {
          wide_store_z<T, VS, ZM>(zl, zv, eb + (e0 + k) * 32, zlv[k]);
          wst(msg + eb + (e0 + k) * 32, gx[k]);
        }
      if (cqt == CB - 1 || c + 1 >= p.n_checks) {
        // End of the item: per-slot partials of its checks (fixed order).
        V* part = reinterpret_cast<V*>(p.part) + ((long long)stripe * ncb + blk) * 64 + lane;
        V a, b;
#pragma unroll
        for (int l = 0; l < VS; ++l) {
          a.v[l] = primal[l];
          b.v[l] = odd[l] ? -moved[l] : moved[l];  // sign bit: an odd check in the block (is_codeword of x_t)
        }
        wst(part, a);
        wst(part + 32, b);
        if (anyret) {
#pragma unroll
          for (int l = 0; l < VS; ++l)
            if (stv.v[l] == kSlotRetiring && odd[l]) atomicOr(p.odd + s0 + l, 1);
        }
#pragma unroll
        for (int l = 0; l < VS; ++l) {
          primal[l] = moved[l] = T(0);
          odd[l] = 0;
        }
      }
    }
  }
  cp_wait<0>();
}

// ---- phase S: one warp per slot ----
template <typename T, int VS>
__device__ __forceinline__ void wide_phase_s(const WideParams<T>& p, int s, int* list, int* nlist) {
  constexpr int W = 32 * VS;
  const int lane = threadIdx.x & 31;
  const int state = __shfl_sync(0xffffffffu, lane == 0 ? p.st[s] : 0, 0);
  if (state == kSlotEmpty) return;
  if (state == kSlotRetiring) {
    if (lane == 0) {
      const long long f = p.frame[s];
      if (p.iters_out) p.iters_out[f] = p.tcount[s];
      if (p.flags_out) p.flags_out[f] = (p.conv[s] ? 1 : 0) | (p.nonint[s] ? 0 : 2) | (p.odd[s] ? 0 : 4);
      if (p.weight_out) p.weight_out[f] = p.weight[s];
      p.tcount[s] = 0;
      p.weight[s] = 0;
      p.nonint[s] = 0;
      p.odd[s] = 0;
      p.conv[s] = 0;
      const int fn = p.fnext[s];
      p.frame[s] = fn;
      if (fn >= 0) {
        p.st[s] = kSlotFresh;
      } else {
        p.st[s] = kSlotEmpty;
        atomicSub(p.ctr + 1, 1);
      }
    }
    return;
  }
  // Exact residual sums (admm_decoder.py:174-176), fixed order; the sign
  // of a moved-partial flags an odd check of x_t in its block.
  const int stripe = s / W, r = s % W;
  const T* part = p.part + (long long)stripe * p.ncb * 2 * W + r;
  // Per-item partials (8 checks) are T; they are accumulated in fp64.
  double a = 0.0, b = 0.0;
  bool odd = false;
#pragma unroll 8
  for (int q = lane; q < p.ncb; q += 32) {
    const T mv = part[(long long)q * 2 * W + W];
    a += static_cast<double>(part[(long long)q * 2 * W]);
    b += static_cast<double>(fabs(mv));
    odd |= signbit(mv);
  }
  a = warp_allsum(a);
  b = warp_allsum(b);
  const bool converged = a < p.thr_d && b < p.thr_d;  // admm_decoder.py:169, 179 (strict)
  const int t = __shfl_sync(0xffffffffu, lane == 0 ? p.tcount[s] : 0, 0) + 1;
  const bool stop = converged || t >= p.t_max;
  if (stop && state == kSlotRunning && p.direct) {
    // Retire now: the outputs of x_t (make_output, :92-105; is_codeword,
    // codes.py:145-154) were accumulated by phases V and C of this pass, and
    // the next frame (popped when this one started) is ready.
    const int n_vb = (p.n_vars + kWideVB - 1) / kWideVB;
    const int* vp = p.vpart + (long long)stripe * n_vb * W + r;
    int w = 0, nonint = 0;
    for (int q = lane; q < n_vb; q += 32) {
      const int v = vp[(long long)q * W];
      w += v & 0xff;
      nonint |= v >> 8;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
    nonint = __any_sync(0xffffffffu, nonint != 0);
    odd = __any_sync(0xffffffffu, odd);
    if (lane == 0) {
      const long long f = p.frame[s];
      if (p.iters_out) p.iters_out[f] = t;
      if (p.flags_out) p.flags_out[f] = (converged ? 1 : 0) | (nonint ? 0 : 2) | (odd ? 0 : 4);
      if (p.weight_out) p.weight_out[f] = w;
      p.tcount[s] = 0;
      const int fn = p.fnext[s];
      p.frame[s] = fn;
      if (fn >= 0) {
        p.st[s] = kSlotFresh;
      } else {
        p.st[s] = kSlotEmpty;
        atomicSub(p.ctr + 1, 1);
      }
    }
    return;
  }
  if (lane == 0) {
    p.tcount[s] = t;
    if (state == kSlotFresh) {
      // The frame that follows this one, popped when this one starts so that
      // (in-kernel synthesis) its LLRs are ready when this one retires.
      const int f = atomicAdd(p.ctr + 0, 1);
      const int fn = f < p.batch ? f : -1;
      p.fnext[s] = fn;
      if (fn >= 0 && p.synth.kind != 0) list[atomicAdd(nlist, 1)] = s;
    }
    if (stop) {
      p.conv[s] = converged;
      p.st[s] = kSlotRetiring;  // the next pass computes the outputs from x_t
    } else {
      p.st[s] = kSlotRunning;
    }
  }
}

// Phase profiler (admm_wide_phase_profile): CTA 0, thread 0 accumulates
// clock64() cycles: 0 step A, 1 sync, 2 slot phase G1 + sync, 3 step B,
// 4 sync, 5 slot phase G0 + sync, 6 passes.
__device__ unsigned long long g_wide_cycles[8];
__device__ int g_wide_prof;

// ctr: [0] frame queue, [1] busy slots, [2] / [3] work items of step A / B,
// [4] / [6] synthesis items of step A / B, [5] / [7] synthesis list lengths
// (list A filled by slot phase G0 for step A, list B by slot phase G1).
template <typename T, int VS, int D, int DVMAX, bool REG, int NS, int MINB>
__global__ void __launch_bounds__(kWideThreads, MINB) wide_decode_kernel(const WideParams<T> p) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) unsigned char wide_smem[];
  constexpr int W = 32 * VS, TS = wide_tstride<D, DVMAX, VS>();
  unsigned char* wbase = wide_smem + (threadIdx.x >> 5) * wide_warp_bytes<T, VS, D, DVMAX, NS>();
  int* tslot = reinterpret_cast<int*>(wbase);
  unsigned char* ring = wbase + 2 * 4 * TS;
  const int n_stripes = p.S / W;
  const int h = (n_stripes + 1) / 2;  // group G0 = stripes [0, h), G1 = [h, n_stripes)
  const int n_vb = (p.n_vars + kWideVB - 1) / kWideVB;
  const int gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int n_gwarp = (gridDim.x * blockDim.x) >> 5;
  const long long first = p.batch < p.S ? p.batch : p.S;
  const bool prof = g_wide_prof && blockIdx.x == 0 && threadIdx.x == 0;
  int* list_a = p.slist;
  int* list_b = p.slist + p.S;
  const bool root = blockIdx.x == 0 && threadIdx.x == 0;

  // Prologue: slot s takes frame s; synthesised LLRs of the first frames.
  if (root) {
    p.ctr[0] = static_cast<int>(first);
    p.ctr[1] = static_cast<int>(first);
    for (int k = 2; k < 8; ++k) p.ctr[k] = 0;
  }
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < p.S; s += gridDim.x * blockDim.x) {
    p.frame[s] = s < first ? s : -1;
    p.st[s] = s < first ? kSlotFresh : kSlotEmpty;
    p.tcount[s] = p.weight[s] = p.nonint[s] = p.odd[s] = p.conv[s] = 0;
  }
  if (p.synth.kind != 0) {
    const long long n = first * p.n_vars;
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n; q += (long long)gridDim.x * blockDim.x)
      p.gfr[q] = static_cast<T>(synth_llr(p.synth, p.synth.trial0 + q / p.n_vars, static_cast<int>(q % p.n_vars)));
  }
  ADMM_JITTER();
  grid.sync();

  const long long max_passes = ((long long)(p.batch + p.S - 1) / p.S + 1) * ((long long)p.t_max + 2) + 4;
  for (long long pass = 0; pass < max_passes; ++pass) {
    if (*(volatile int*)(p.ctr + 1) == 0) break;
    long long tp[7];
    tp[0] = prof ? clock64() : 0;
    // step A: phase V of G0, phase C of G1 (G1 has no x yet in the first pass)
    if (p.synth.kind != 0) wide_synth_items(p, list_a, *(volatile int*)(p.ctr + 5), p.ctr + 4);
    {
      const WideStep sa(0, h, h, pass == 0 ? 0 : n_stripes - h, n_vb, p.ncb);
      wide_step<T, VS, D, DVMAX, REG, NS>(p, ring, tslot, TS, sa, p.ctr + 2);
    }
    if (prof) tp[1] = clock64();
    ADMM_JITTER();
    grid.sync();
    if (prof) tp[2] = clock64();
    // slot phase of G1; reset the counters step B will use and list A
    if (root) {
      p.ctr[3] = 0;
      p.ctr[6] = 0;
      p.ctr[5] = 0;
    }
    if (pass > 0)
      for (int s = h * W + gwarp; s < p.S; s += n_gwarp) wide_phase_s<T, VS>(p, s, list_b, p.ctr + 7);
    ADMM_JITTER();
    grid.sync();
    if (prof) tp[3] = clock64();
    // step B: phase C of G0, phase V of G1
    if (p.synth.kind != 0) wide_synth_items(p, list_b, *(volatile int*)(p.ctr + 7), p.ctr + 6);
    {
      const WideStep sb(h, n_stripes - h, 0, h, n_vb, p.ncb);
      wide_step<T, VS, D, DVMAX, REG, NS>(p, ring, tslot, TS, sb, p.ctr + 3);
    }
    if (prof) tp[4] = clock64();
    ADMM_JITTER();
    grid.sync();
    if (prof) tp[5] = clock64();
    // slot phase of G0; reset the counters step A will use and list B
    if (root) {
      p.ctr[2] = 0;
      p.ctr[4] = 0;
      p.ctr[7] = 0;
    }
    for (int s = gwarp; s < h * W; s += n_gwarp) wide_phase_s<T, VS>(p, s, list_a, p.ctr + 5);
    ADMM_JITTER();
    grid.sync();
    if (prof) {
      tp[6] = clock64();
#pragma unroll
      for (int k = 0; k < 6; ++k) g_wide_cycles[k] += tp[k + 1] - tp[k];
      g_wide_cycles[6] += 1;
    }
  }
}

}  // namespace admm
