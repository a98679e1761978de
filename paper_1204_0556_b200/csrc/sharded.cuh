// Sharded streaming engine: the streaming engine's slot machine (streaming.cuh)
// with a STATIC partition of the Tanner graph over the persistent CTAs.
//
// CTA b owns checks [b*MB, (b+1)*MB) and variables [b*NB, (b+1)*NB) for all
// S frame slots.  Because the assignment never changes, the replicas z and
// duals lambda of its checks' edges stay in the CTA's SHARED MEMORY for the
// whole run ([edge][slot] pairs), next to gamma/mu of its variables and the
// graph indices of both; only the messages z - lambda/mu and the variables x
// ([edge][slot] / [var][slot], slot-minor, so every warp access is 32
// consecutive slots = 128 B) cross the chip through L2:
//     phase V  reads 3 messages, writes x          (~5.3 B per edge-update)
//     phase C  gathers x, writes the message       (~8 B per edge-update)
// versus ~31 B per edge-update when z and lambda also stream through memory.
// Duals are kept scaled (lambda / mu, the reference's message-passing form).
// The cross-CTA gathers use ld.global.cg: with ~205 KB of the unified L1 given
// to shared memory, L1-allocating loads can only keep ~150 line misses in
// flight per SM, while L2-only loads keep the whole batch in flight (an L2
// round trip under full load is ~2.7k cycles, tools/micro/l2mlp.cu).
//
// Slot management is REPLICATED: every CTA keeps the slot states, iteration
// counters and frame indices in its own shared memory and takes the same
// decisions from the same global inputs (the per-slot not-converged flags and
// the fixed-order partial sums), refilling retired slots in slot order from a
// replicated frame counter.  An iteration therefore needs two grid syncs
// (after the variable phase and after the check phase), not three.
// Partial residual sums are accumulated per lane (one slot) over the warp's
// checks in a fixed order and combined per slot across warps and CTAs in a
// fixed order, so the stop decision is deterministic.
#pragma once

#include "streaming.cuh"

namespace admm {

// One CTA per SM: 32 warps in fp32 (64 registers fit), 16 in fp64 (the
// double-precision check update needs ~110 registers; at 64 it spills).
template <typename T> struct ShardThreads { static constexpr int value = sizeof(T) == 4 ? 1024 : 512; };
constexpr int kShardThreadsMax = 1024;

// Phase profiler (admm_phase_profile): CTA 0, thread 0 accumulates clock64()
// cycles per phase when enabled.  Slots: 0 variable phase, 1 grid sync after
// it, 2 check phase, 3 grid sync after it, 4 slot phase, 5 passes.
__device__ unsigned long long g_phase_cycles[8];
__device__ int g_phase_on;

struct ShardGeom {
  int MB, NB, EB;  // checks, variables, edges (max) per CTA
  int zl, gm, cv, ce, ve, red, sint, slot, total;  // shared-memory offsets (bytes)
};

inline ShardGeom shard_geom(int elem, int D, int dvmax, int M, int N, long long max_edges_per_cta, int G, int S) {
  ShardGeom g{};
  g.MB = (M + G - 1) / G;
  g.NB = (N + G - 1) / G;
  g.EB = static_cast<int>(max_edges_per_cta);
  auto al = [](long long b) { return static_cast<int>((b + 15) & ~15ll); };
  int o = 0;
  g.zl = o; o = al(o + 2ll * elem * g.EB * S);
  g.gm = o; o = al(o + 1ll * elem * g.NB * S);
  g.cv = o; o = al(o + 4ll * g.MB * D);
  g.ce = o; o = al(o + 4ll * g.MB);
  g.ve = o; o = al(o + 4ll * g.NB * dvmax);
  g.red = o; o = al(o + 2ll * elem * (kShardThreadsMax / 32) * 32);
  g.sint = o; o = al(o + 4ll * 2 * S);
  g.slot = o; o = al(o + 8ll * S + 4ll * 4 * S + 4 * (4 + 32) + 16);  // replicated slot machine
  g.total = o;
  return g;
}

template <typename T, int D, int DVMAX, bool REG>
__global__ void __launch_bounds__(ShardThreads<T>::value, 1) sharded_decode_kernel(const StreamParams<T> p, const ShardGeom geo) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, nwarps = blockDim.x >> 5;
  const int S = p.S, SG = S / 32, NWG = nwarps / SG;
  const int b = blockIdx.x, G = gridDim.x;
  const int cb0 = b * geo.MB, cb1 = min(p.n_checks, cb0 + geo.MB);
  const int vb0 = b * geo.NB, vb1 = min(p.n_vars, vb0 + geo.NB);
  const int mb = max(0, cb1 - cb0), nb = max(0, vb1 - vb0);
  T* zl_s = reinterpret_cast<T*>(smem_raw + geo.zl);  // [edge - eb0][S][2]
  T* gm_s = reinterpret_cast<T*>(smem_raw + geo.gm);  // [var - vb0][S]
  // Graph slice, stored pre-multiplied by S (element offsets of slot 0), -1 = unused.
  int* cv_s = reinterpret_cast<int*>(smem_raw + geo.cv);  // [check - cb0][D]    var * S
  int* ce_s = reinterpret_cast<int*>(smem_raw + geo.ce);  // [check - cb0]       (local edge) * S
  int* ve_s = reinterpret_cast<int*>(smem_raw + geo.ve);  // [var - vb0][DVMAX]  (global edge) * S
  T* red = reinterpret_cast<T*>(smem_raw + geo.red);      // [16][32][2]
  int* sint = reinterpret_cast<int*>(smem_raw + geo.sint);  // [S] weight, [S] non-integral (retiring)
  const long long eb0 = mb > 0 ? __ldg(p.edge_base + cb0) : 0;

  // ---- static graph slice (once) ----
  for (int q = tid; q < mb * D; q += blockDim.x) {
    const int lc = q / D, k = q % D;
    const int v = __ldg(p.chk_var + k * p.m_pad + cb0 + lc);
    cv_s[q] = v >= 0 ? v * S : -1;
  }
  for (int q = tid; q < mb; q += blockDim.x) ce_s[q] = static_cast<int>(__ldg(p.edge_base + cb0 + q) - eb0) * S;
  for (int q = tid; q < nb * DVMAX; q += blockDim.x) {
    const int lv = q / DVMAX, j = q % DVMAX;
    const int e = j < p.dvmax ? __ldg(p.var_edge + (vb0 + lv) * p.dvmax + j) : -1;
    ve_s[q] = e >= 0 ? e * S : -1;
  }
  // ---- replicated slot machine (shared memory, identical in every CTA) ----
  long long* fr_s = reinterpret_cast<long long*>(smem_raw + geo.slot);  // [S] frame
  int* st_s = reinterpret_cast<int*>(fr_s + S);                         // [S] state
  int* t_s = st_s + S;                                                  // [S] iterations
  int* cv_f = t_s + S;                                                  // [S] converged (retiring)
  int* dec_s = cv_f + S;                                                // [S] decision scratch
  int* misc = dec_s + S;  // [0] active slots, [2..3] next frame (int64), [4..35] warp scan
  // not-converged flags, double-buffered by pass parity; slot s at [32 s] so
  // the ~G atomics per slot and pass land on distinct L2 lines
  int* ncb[2] = {p.flagpad, p.flagpad + 32 * S};
  for (int s = tid; s < S; s += blockDim.x) {
    const long long f = s;
    fr_s[s] = f < p.batch ? f : -1;
    st_s[s] = f < p.batch ? kSlotFresh : kSlotEmpty;
    t_s[s] = 0;
    cv_f[s] = 0;
    if (b == 0) {
      ncb[0][32 * s] = 0;
      ncb[1][32 * s] = 0;
      p.weight[s] = 0;
      p.nonint[s] = 0;
      p.odd[s] = 0;
    }
  }
  if (tid == 0) {
    const long long first = p.batch < S ? p.batch : S;
    misc[0] = static_cast<int>(first);
    *reinterpret_cast<long long*>(misc + 2) = first;
  }
  ADMM_JITTER();
  grid.sync();

  const long long max_passes = ((long long)(p.batch + S - 1) / S + 1) * ((long long)p.t_max + 2) + 4;
  for (long long pass = 0; pass < max_passes; ++pass) {
    __syncthreads();
    if (misc[0] == 0) break;
    int* nc_now = ncb[pass & 1];

    const bool prof = g_phase_on && b == 0 && tid == 0;
    long long tp0 = prof ? clock64() : 0;
    const long long SS = S;
    // ---------------- phase V: this CTA's variables, all slots ----------------
    for (int q = tid; q < 2 * S; q += blockDim.x) sint[q] = 0;
    __syncthreads();
    long long tpa = prof ? clock64() : 0;
    {
      const int sg = w & (SG - 1), wi = w / SG;  // SG is a power of two
      const int s = sg * 32 + lane;
      const int state = st_s[s];
      const long long f = fr_s[s];
      T* xcol = p.x + s;
      const T* mcol = p.msg + s;
      // Batches of VB variables: every global load of a batch (messages of
      // RUNNING slots, gamma or synthesis of FRESH slots, the final x of
      // RETIRING slots) is issued before any is consumed.
      constexpr int VB = 4;
      if (state == kSlotRetiring) {
        for (int lv0 = wi; lv0 < nb; lv0 += VB * NWG) {
          T xq[VB];
#pragma unroll
          for (int q = 0; q < VB; ++q) {
            const int lv = lv0 + q * NWG;
            xq[q] = lv < nb ? __ldcg(xcol + (vb0 + lv) * S) : T(0);
          }
#pragma unroll
          for (int q = 0; q < VB; ++q) {
            const int lv = lv0 + q * NWG;
            if (lv >= nb) break;
            const int i = vb0 + lv;
            const T xv = xq[q];
            const bool h = xv > T(0.5);
            if (p.x_out) p.x_out[f * p.ld_x + i] = xv;
            if (p.hard_out) p.hard_out[f * p.ld_hard + i] = h;
            if (h) atomicAdd_block(sint + s, 1);
            if (!(vmin(fabs(xv), fabs(T(1) - xv)) <= T(1e-5))) atomicOr_block(sint + S + s, 1);
          }
        }
      } else if (state != kSlotEmpty) {
        const bool fresh = state == kSlotFresh;
        long long tq0 = prof ? clock64() : 0;
        for (int lv0 = wi; lv0 < nb; lv0 += VB * NWG) {
          T mv[VB][DVMAX];
          T gq[VB];
          int degs[VB];
#pragma unroll
          for (int q = 0; q < VB; ++q) {
            const int lv = lv0 + q * NWG;
            const bool inb = lv < nb;
            degs[q] = 0;
#pragma unroll
            for (int j = 0; j < DVMAX; ++j) {
              const int ev = inb ? ve_s[lv * DVMAX + j] : -1;
              degs[q] += ev >= 0;
              mv[q][j] = (ev >= 0 && !fresh) ? __ldcg(mcol + ev) : T(0);
            }
            if (!inb) {
              gq[q] = T(0);
            } else if (!fresh) {
              gq[q] = gm_s[lv * S + s];
            } else {
              const int i = vb0 + lv;
              gq[q] = p.synth.kind != 0 ? static_cast<T>(synth_llr(p.synth, p.synth.trial0 + f, i))
                                        : p.gamma[f * p.ld_gamma + i];
            }
          }
#pragma unroll
          for (int q = 0; q < VB; ++q) {
            const int lv = lv0 + q * NWG;
            if (lv >= nb) break;
            const int i = vb0 + lv;
            T g = gq[q];
            if (fresh) {
              g = div_rn(g, p.mu);
              gm_s[lv * S + s] = g;
            }
            const int deg = REG ? DVMAX : degs[q];
            T acc = T(0);
#pragma unroll
            for (int j = 0; j < DVMAX; ++j)
              if (REG || j < deg) acc = add_rn(acc, mv[q][j]);  // unused slots are 0 and at the end
            T xv;
            if (REG || deg > 0) {
              const T num = sub_rn(acc, g);
              const T inv = REG ? T(1) / T(DVMAX) : T(1) / T(deg);
              xv = clip01(mul_rn(num, inv));
            } else {
              xv = g < T(0) ? T(1) : T(0);
            }
            xcol[i * S] = xv;
          }
          if (prof && lv0 == wi) {
            g_phase_cycles[6] += clock64() - tq0;  // first batch: loads issued and consumed
            g_phase_cycles[7] += 1;
          }
        }
      }
    }
    long long tpb = prof ? clock64() : 0;
    (void)tpa;
    (void)tpb;
    __syncthreads();
    for (int s = tid; s < S; s += blockDim.x) {
      if (sint[s]) atomicAdd(p.weight + s, sint[s]);
      if (sint[S + s]) atomicOr(p.nonint + s, 1);
    }
    long long tp1 = prof ? clock64() : 0;
    ADMM_JITTER();
    grid.sync();
    long long tp2 = prof ? clock64() : 0;

    // ---------------- phase C: this CTA's checks, all slots ----------------
    if (b == 0)  // the other flag buffer was last read in the previous pass's slot phase
      for (int q = tid; q < S; q += blockDim.x) ncb[(pass + 1) & 1][32 * q] = 0;
    {
      const int sg = w % SG, wi = w / SG;
      const int s = sg * 32 + lane;
      const int state = st_s[s];
      const bool live = state == kSlotFresh || state == kSlotRunning;
      T primal = T(0), moved = T(0);
      int odd = 0;
      if (live || state == kSlotRetiring) {
        const T* xcol = p.x + s;
        T* mcol = p.msg + s;
        T* zcol = zl_s + 2 * s;
        const long long geS = eb0 * S;
        // Software pipeline: the x-gathers of the warp's next check are in
        // flight while the current check is projected.
        T gx_nx[D];
        int d_nx = D;
        auto gather = [&](int lc, T (&dst)[D], int& dd) {
          int vo[D];
#pragma unroll
          for (int k = 0; k < D; ++k) vo[k] = cv_s[lc * D + k];
          dd = D;
          if (!REG) {
            dd = 0;
#pragma unroll
            for (int k = 0; k < D; ++k) dd += vo[k] >= 0;
          }
#pragma unroll
          for (int k = 0; k < D; ++k) dst[k] = (REG || k < dd) ? __ldcg(xcol + vo[k]) : T(0);
        };
        if (wi < mb) gather(wi, gx_nx, d_nx);
        for (int lc = wi; lc < mb; lc += NWG) {
          T gx[D];
#pragma unroll
          for (int k = 0; k < D; ++k) gx[k] = gx_nx[k];
          const int d = d_nx;
          if (lc + NWG < mb) gather(lc + NWG, gx_nx, d_nx);
          if (!live) {  // retiring: syndrome of the final hard decision (codes.py:145-154)
            int par = 0;
#pragma unroll
            for (int k = 0; k < D; ++k)
              if (REG || k < d) par ^= gx[k] > T(0.5);
            odd |= par;
            continue;
          }
          const int le = ce_s[lc];  // (local edge) * S
          T z[D], lam[D], w_[D], u[D], zn[D];
#pragma unroll
          for (int k = 0; k < D; ++k) {
            z[k] = T(0);
            lam[k] = T(0);
            if ((REG || k < d) && state == kSlotRunning) {
              const T* zp = zcol + 2 * (le + k * S);
              z[k] = zp[0];
              lam[k] = zp[1];
            }
            w_[k] = add_rn(mul_rn(p.rho, gx[k]), mul_rn(p.one_minus_rho, z[k]));
            u[k] = (REG || k < d) ? add_rn(w_[k], lam[k]) : -Num<T>::inf();  // lam holds lambda/mu
          }
          if constexpr (REG) {
            project_pp_fixed<T, D>(u, zn);
          } else {
            project_pp<T, D>(u, zn, d);
          }
#pragma unroll
          for (int k = 0; k < D; ++k) {
            if (REG || k < d) {
              const T r1 = sub_rn(gx[k], zn[k]);
              const T r2 = sub_rn(zn[k], z[k]);
              primal = add_rn(primal, mul_rn(r1, r1));
              moved = add_rn(moved, mul_rn(r2, r2));
              const T lnew = add_rn(lam[k], sub_rn(w_[k], zn[k]));  // scaled dual lambda/mu
              T* zp = zcol + 2 * (le + k * S);
              zp[0] = zn[k];
              zp[1] = lnew;
              mcol[geS + le + k * S] = sub_rn(zn[k], lnew);
            }
          }
        }
      }
      // Per-slot partials over the CTA's checks: warps of one slot group in a
      // fixed order.
      red[(w * 32 + lane) * 2] = live ? primal : T(odd);
      red[(w * 32 + lane) * 2 + 1] = moved;
      __syncthreads();
      if (wi == 0) {
        T a = T(0), bb = T(0);
        for (int q = 0; q < NWG; ++q) {
          const int ww = q * SG + sg;
          a = add_rn(a, red[(ww * 32 + lane) * 2]);
          bb = add_rn(bb, red[(ww * 32 + lane) * 2 + 1]);
        }
        if (live) {
          p.part[((long long)b * S + s) * 2] = a;
          p.part[((long long)b * S + s) * 2 + 1] = bb;
          if (a >= p.thr || bb >= p.thr) atomicOr(nc_now + 32 * s, 1);
        } else if (state == kSlotRetiring && a > T(0)) {
          atomicOr(p.odd + s, 1);
        }
      }
    }
    long long tp3 = prof ? clock64() : 0;
    ADMM_JITTER();
    grid.sync();
    long long tp4 = prof ? clock64() : 0;

    // ---------------- phase S: replicated in every CTA (no grid sync) ----------------
    // (a) exact residual sums for the slots whose every partial is below the
    //     threshold (admm_decoder.py:174-179): one warp per slot, fixed tree.
    //     The flags are fetched for all slots at once first.
    for (int q = tid; q < S; q += blockDim.x) dec_s[q] = nc_now[32 * q];
    __syncthreads();
    for (int q = w; q < S; q += nwarps) {
      const int state = st_s[q];
      int conv = 0;
      if ((state == kSlotFresh || state == kSlotRunning) && dec_s[q] == 0) {
        double a = 0.0, bb = 0.0;  // per-CTA partials accumulated in fp64
        for (int r = lane; r < G; r += 32) {
          a += static_cast<double>(p.part[((long long)r * S + q) * 2]);
          bb += static_cast<double>(p.part[((long long)r * S + q) * 2 + 1]);
        }
        a = warp_allsum(a);
        bb = warp_allsum(bb);
        conv = a < p.thr_d && bb < p.thr_d;
      }
      __syncwarp();
      if (lane == 0) dec_s[q] = conv;
    }
    __syncthreads();
    // (b) state transitions; retired slots are refilled in slot order from the
    //     replicated frame counter (a block-wide scan gives each its rank).
    long long* next = reinterpret_cast<long long*>(misc + 2);
    int* wscan = misc + 4;
    for (int s0 = 0; s0 < S; s0 += blockDim.x) {
      const int q = s0 + tid;
      const int state = q < S ? st_s[q] : kSlotEmpty;
      const bool retiring = state == kSlotRetiring;
      if (q < S && retiring && b == 0) {
        const long long f = fr_s[q];
        if (p.iters_out) p.iters_out[f] = t_s[q];
        if (p.flags_out) p.flags_out[f] = (cv_f[q] ? 1 : 0) | (p.nonint[q] ? 0 : 2) | (p.odd[q] ? 0 : 4);
        if (p.weight_out) p.weight_out[f] = p.weight[q];
        p.weight[q] = 0;
        p.nonint[q] = 0;
        p.odd[q] = 0;
      }
      if (q < S && (state == kSlotFresh || state == kSlotRunning)) {
        const int t = t_s[q] + 1;
        t_s[q] = t;
        if (dec_s[q] || t >= p.t_max) {
          cv_f[q] = dec_s[q];
          st_s[q] = kSlotRetiring;
        } else {
          st_s[q] = kSlotRunning;
        }
      }
      const unsigned bal = __ballot_sync(0xffffffffu, retiring);
      if (lane == 0) wscan[w] = __popc(bal);
      __syncthreads();
      int before = 0, total = 0;
      for (int ww = 0; ww < nwarps; ++ww) {
        before += ww < w ? wscan[ww] : 0;
        total += wscan[ww];
      }
      const long long base = *next;
      if (retiring) {
        const long long f = base + before + __popc(bal & ((1u << lane) - 1u));
        t_s[q] = 0;
        cv_f[q] = 0;
        if (f < p.batch) {
          fr_s[q] = f;
          st_s[q] = kSlotFresh;
        } else {
          fr_s[q] = -1;
          st_s[q] = kSlotEmpty;
          atomicSub_block(misc, 1);
        }
      }
      __syncthreads();
      if (tid == 0) *next = base + total;
    }
    if (prof) {
      const long long tp5 = clock64();
      g_phase_cycles[0] += tp1 - tp0;
      g_phase_cycles[1] += tp2 - tp1;
      g_phase_cycles[2] += tp3 - tp2;
      g_phase_cycles[3] += tp4 - tp3;
      g_phase_cycles[4] += tp5 - tp4;
      g_phase_cycles[5] += 1;
    }
    // No grid sync here: every cross-CTA read of the next pass is separated
    // from the last write it depends on by the sync after its variable phase
    // (p.part, the flag buffers, the weight/odd/non-integral counters of the
    // slots that retired in this pass) or after this pass's check phase
    // (messages, x).
  }
}

}  // namespace admm
