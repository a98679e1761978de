// Host-side layout of the cluster engine (cluster.cuh): one thread-block
// cluster of C CTAs decodes one frame, CTA ("part") p owning M/C checks and
// N/C variables.
//
// Partition.  The checks are split into C balanced parts so that few
// variables have checks in more than one part (hypergraph partitioning:
// checks are vertices, variables are nets, minimise the connectivity
// sum_v (|P(v)| - 1) where P(v) is the set of parts holding v's checks).
// Each variable is then OWNED by the part holding most of its checks and is a
// GHOST in the other parts of P(v).  Per iteration a part ships (a) the x of
// its owned variables to every part that holds them as ghosts and (b) the
// messages of its checks' edges to ghost variables to their owners -- both
// ~ the connectivity, ~2.8k values each per part on config 5 (C = 4).
// DSMEM prices scattered 4-byte remote accesses at ~2.6 SM cycles each but
// moves warp-coalesced stores at ~20-25 B/cycle (tools/micro/dsmem.cu), so
// every exchange is table-driven: a warp gathers 32 local values and stores
// them to 32 CONSECUTIVE words of the destination.  For the x-send that is
// the destination's ghost region (ordered like the sender's list); for the
// messages it is the owner's message rows THEMSELVES: the owner's variables
// are ordered by their edge signature (the part holding each color's edge),
// so the messages one part sends for one color land in a few long runs of
// consecutive own slots -- no inbox and no scatter on the receiving side.
// Simulated annealing over check swaps between parts (balance is kept
// exactly), from a BFS-grown initial partition.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <deque>
#include <random>
#include <string>
#include <utility>
#include <vector>

#include "layout.h"

namespace admm {

// Packed message-table entry: color j (2 bits) | ghost slot in the sender
// (13) | own slot in the owner (12) | owner rank (3) -- shared with cluster.cuh.
inline constexpr uint32_t ms_entry(uint32_t j, uint32_t gslot, uint32_t oslot, uint32_t rank) {
  return j | gslot << 2 | oslot << 15 | rank << 27;
}

struct ClusterPartition {
  int C = 0;
  std::vector<int> part_of_check;  // [M]
  long long connectivity = 0;      // sum_v (|P(v)| - 1)
  long long exchange = 0;          // messages shipped per iteration (all parts)
  long long replicas = 0;          // sum_v |P(v)| (local variables over all parts)
};

// Exchange volume of variable v given its per-part edge counts, owned by the
// part with most of its edges: (|P(v)| - 1) ghost x values plus the messages
// of its edges outside the owner.
inline long long var_exchange(const int* cnt, int C) {
  int lam = 0, deg = 0, mx = 0;
  for (int p = 0; p < C; ++p) {
    lam += cnt[p] > 0;
    deg += cnt[p];
    mx = cnt[p] > mx ? cnt[p] : mx;
  }
  return lam > 0 ? static_cast<long long>(lam - 1) + (deg - mx) : 0;
}

inline ClusterPartition partition_checks(const std::vector<std::vector<int>>& rows, int n_vars, int C,
                                         long long moves, uint64_t seed) {
  const int M = static_cast<int>(rows.size());
  ClusterPartition P;
  P.C = C;
  std::mt19937_64 rng(seed);
  std::vector<std::vector<int>> var_checks(n_vars);
  for (int c = 0; c < M; ++c)
    for (int v : rows[c]) var_checks[v].push_back(c);
  // Balanced part sizes (differ by at most one).
  std::vector<int> cap(C);
  for (int p = 0; p < C; ++p) cap[p] = M / C + (p < M % C ? 1 : 0);
  // Initial partition: grow each part by BFS over the check-variable-check
  // graph from a random unassigned seed check.
  P.part_of_check.assign(M, -1);
  {
    std::vector<int> order(M);
    for (int c = 0; c < M; ++c) order[c] = c;
    std::shuffle(order.begin(), order.end(), rng);
    size_t oi = 0;
    for (int p = 0; p < C; ++p) {
      int filled = 0;
      std::deque<int> q;
      while (filled < cap[p]) {
        if (q.empty()) {
          while (oi < order.size() && P.part_of_check[order[oi]] >= 0) ++oi;
          if (oi == order.size()) break;
          q.push_back(order[oi]);
          P.part_of_check[order[oi]] = p;
          ++filled;
        }
        const int c = q.front();
        q.pop_front();
        for (int v : rows[c])
          for (int c2 : var_checks[v])
            if (P.part_of_check[c2] < 0 && filled < cap[p]) {
              P.part_of_check[c2] = p;
              ++filled;
              q.push_back(c2);
            }
      }
    }
  }
  // cnt[v][p]: edges of v in part p.
  std::vector<int> cnt(static_cast<size_t>(n_vars) * C, 0);
  for (int c = 0; c < M; ++c)
    for (int v : rows[c]) cnt[static_cast<size_t>(v) * C + P.part_of_check[c]]++;
  std::vector<std::vector<int>> members(C);
  std::vector<int> pos(M);
  for (int c = 0; c < M; ++c) {
    pos[c] = static_cast<int>(members[P.part_of_check[c]].size());
    members[P.part_of_check[c]].push_back(c);
  }
  long long cost = 0;
  for (int v = 0; v < n_vars; ++v) cost += var_exchange(&cnt[static_cast<size_t>(v) * C], C);
  // move c from part a to part b: change of the exchange volume
  auto move = [&](int c, int a, int b) {
    long long d = 0;
    for (int v : rows[c]) {
      int* k = &cnt[static_cast<size_t>(v) * C];
      d -= var_exchange(k, C);
      k[a]--;
      k[b]++;
      d += var_exchange(k, C);
    }
    return d;
  };
  std::uniform_real_distribution<double> U(0.0, 1.0);
  double T = 2.0;
  const double decay = std::pow(0.01 / T, 1.0 / static_cast<double>(std::max<long long>(1, moves)));
  for (long long it = 0; it < moves; ++it, T *= decay) {
    // a check next to the boundary, moved towards a part one of its variables touches
    const int c = static_cast<int>(rng() % M);
    const int a = P.part_of_check[c];
    const int v = rows[c][rng() % rows[c].size()];
    const std::vector<int>& vc = var_checks[v];
    const int b = P.part_of_check[vc[rng() % vc.size()]];
    if (a == b) continue;
    const int c2 = members[b][rng() % members[b].size()];
    long long d = move(c, a, b);
    d += move(c2, b, a);
    if (d <= 0 || U(rng) < std::exp(-static_cast<double>(d) / T)) {
      cost += d;
      P.part_of_check[c] = b;
      P.part_of_check[c2] = a;
      members[b][pos[c2]] = c;
      members[a][pos[c]] = c2;
      std::swap(pos[c], pos[c2]);
    } else {
      move(c2, a, b);
      move(c, b, a);
    }
  }
  P.exchange = cost;
  P.connectivity = 0;
  P.replicas = 0;
  for (int v = 0; v < n_vars; ++v) {
    int lam = 0;
    for (int p = 0; p < C; ++p) lam += cnt[static_cast<size_t>(v) * C + p] > 0;
    P.connectivity += lam > 0 ? lam - 1 : 0;
    P.replicas += lam;
  }
  return P;
}

// ---------------------------------------------------------------------------
// Per-part slot layout and exchange tables.
//
// Shared memory of part p (fp32 words): X[NPL] | MSG[DV][NPL] | GM[NPL] | ...
// (row j of the messages starts at word (j + 1) NPL)
//   local slots [0, NO)            the part's OWN variables (NO = NT * VPT;
//                                  thread t owns slots 2t, 2t+1, 2t+2NT, ...)
//   [NO, NO + ghosts)              GHOST variables, grouped by owner part o
//                                  at gbase[p][o] (x written by o each pass)
//   NO + ghosts                    spare slot (idle checks gather / write it)
// The message of edge (c, v) of color j (equitable coloring of layout.h:
// every variable has one edge per color, slot k of a check has color k % DV)
// lives at MSG[j][slot(v)]: for own v it is consumed by the variable phase,
// for a ghost v it is shipped (msend table) to MSG[j][own slot of v] of the
// owner.
struct ClusterLayout {
  int C = 0, NT = 0, CPT = 0, VPT = 0, D = 0, DV = 0;
  int MC = 0;   // local check slots per part (NT * CPT)
  int NO = 0;   // own variable slots per part (NT * VPT)
  int NPL = 0;  // local slots per part (own + ghosts + spare), multiple of 32
  int NXS = 0, NMS = 0;  // table capacities (max over parts), multiples of 32
  std::vector<int> chk_slot;        // [C][D][MC] local slot of the variable in slot k of local check lc
  std::vector<int> chk_orig;        // [C][MC] original check (-1: idle)
  std::vector<int> own_var;         // [C][NO] original variable of an own slot (-1: dummy)
  std::vector<int> xs_start;        // [C][C+1] xsend range of part p for destination r: [xs_start[p][r], xs_start[p][r+1])
  std::vector<int> gbase;           // [C][C] gbase[r][o]: first ghost slot in part r of the variables owned by o
  std::vector<int> n_ms;            // [C] msend entries of part p
  std::vector<int> nb;              // [C] own slots [0, nb) hold the boundary variables; the kernel
                                    // updates the pairs starting below nb first
  std::vector<int> nic;             // [C] local check slots [0, nic) hold the interior checks
  std::vector<uint16_t> xsend;      // [C][NXS] own slots whose x goes to ghosts (grouped by destination)
  std::vector<uint32_t> msend;      // [C][NMS] ms_entry(color, ghost slot here, own slot at the owner, owner)
  ClusterPartition part;
  long long ghost_total = 0, msg_total = 0;
  int msg_runs = 0;                 // maximal runs of consecutive destination words (all parts)
  double bank_cost_before = 0, bank_cost_after = 0;
  bool ok = false;
  std::string error;
};

inline ClusterLayout build_cluster_layout(const std::vector<std::vector<int>>& rows, int n_vars, int D, int DV,
                                          int C, int NT, int CPT, int VPT, long long part_moves,
                                          long long bank_moves, uint64_t seed) {
  ClusterLayout L;
  L.C = C, L.NT = NT, L.CPT = CPT, L.VPT = VPT, L.D = D, L.DV = DV;
  L.MC = NT * CPT;
  L.NO = NT * VPT;
  const int M = static_cast<int>(rows.size());
  for (const auto& r : rows)
    if (static_cast<int>(r.size()) != D) {
      L.error = "cluster engine: check-regular codes only";
      return L;
    }
  if ((M + C - 1) / C > L.MC) {
    L.error = "cluster engine: too many checks per part";
    return L;
  }
  // equitable coloring (slot k of a check has color k % DV)
  const Layout col = optimize_colored_layout(rows, n_vars, D, DV, 0, seed);
  if (col.clashes || D % DV != 0) {
    L.error = "cluster engine: no equitable edge coloring";
    return L;
  }
  L.part = partition_checks(rows, n_vars, C, part_moves, seed + 1);
  const std::vector<int>& pc = L.part.part_of_check;
  std::vector<int> cnt(static_cast<size_t>(n_vars) * C, 0);
  for (int c = 0; c < M; ++c)
    for (int v : rows[c]) cnt[static_cast<size_t>(v) * C + pc[c]]++;
  // Ownership: the part with most of the variable's edges; then balance to
  // at most NO per part, moving ties first (no extra exchange), then 2+1 splits.
  std::vector<int> owner(n_vars, -1), owned(C, 0);
  for (int v = 0; v < n_vars; ++v) {
    int best = -1;
    for (int p = 0; p < C; ++p) {
      const int k = cnt[static_cast<size_t>(v) * C + p];
      if (k == 0) continue;
      if (best < 0 || k > cnt[static_cast<size_t>(v) * C + best] ||
          (k == cnt[static_cast<size_t>(v) * C + best] && owned[p] < owned[best]))
        best = p;
    }
    if (best < 0) best = static_cast<int>(std::min_element(owned.begin(), owned.end()) - owned.begin());  // degree 0
    owner[v] = best;
    owned[best]++;
  }
  for (int pass = 0; pass < 3; ++pass) {
    for (int v = 0; v < n_vars; ++v) {
      const int a = owner[v];
      if (owned[a] <= L.NO) continue;
      const int* k = &cnt[static_cast<size_t>(v) * C];
      int best = -1;
      for (int b = 0; b < C; ++b) {
        if (b == a || owned[b] >= L.NO) continue;
        const bool ok = pass == 0 ? (k[b] > 0 && k[b] == k[a]) : pass == 1 ? k[b] > 0 : true;
        if (ok && (best < 0 || k[b] > k[best])) best = b;
      }
      if (best >= 0) {
        owner[v] = best;
        owned[a]--;
        owned[best]++;
      }
    }
  }
  for (int p = 0; p < C; ++p)
    if (owned[p] > L.NO) {
      L.error = "cluster engine: variable ownership does not balance";
      return L;
    }
  // A variable is BOUNDARY if it has edges in more than one part (its x is
  // shipped to ghosts, its owner receives messages); a check is INTERIOR if
  // none of its variables is a ghost in its part.  Boundary own variables take
  // the first own slots [0, nb) (nb even: variable pairs), interior checks the
  // first local check slots [0, nic): the kernel updates boundary variables
  // first, ships their x, and overlaps the cluster barrier with the interior
  // variables and checks (cluster.cuh).  (nb may be odd: the pair straddling
// it is updated with the boundary pairs.)
  std::vector<char> boundary(n_vars, 0);
  for (int v = 0; v < n_vars; ++v) {
    int lam = 0;
    for (int p = 0; p < C; ++p) lam += cnt[static_cast<size_t>(v) * C + p] > 0;
    boundary[v] = lam > 1;
  }
  std::vector<std::vector<int>> pchecks(C);
  L.nic.assign(C, 0);
  for (int pass = 0; pass < 2; ++pass)
    for (int c = 0; c < M; ++c) {
      bool interior = true;
      for (int v : rows[c]) interior &= owner[v] == pc[c];
      if (interior == (pass == 0)) {
        pchecks[pc[c]].push_back(c);
        L.nic[pc[c]] += interior;
      }
    }
  // Own slots: owned variables sorted by their edge signature (the part of
  // the color-0, -1, -2 edge), so that the messages part q sends to part o
  // for color j land in runs of consecutive own slots of o; ties in index
  // order (the bank annealer permutes slots inside a signature class).
  std::vector<int> sig(n_vars, 0);
  for (int c = 0; c < M; ++c)
    for (int r = 0; r < D; ++r) {
      const int j = col.edge_slot[c * D + r] % DV, v = rows[c][r];
      int w = 1;
      for (int i = j + 1; i < DV; ++i) w *= C;
      sig[v] += pc[c] * w;
    }
  std::vector<std::vector<int>> slot_var(C);  // [p][slot] -> variable (-1 dummy / spare)
  std::vector<std::vector<int>> ghosts_of(C * C);  // [r][o] ghost variables of part r owned by o
  std::vector<std::vector<int>> slot_class(C);  // [p][own slot] signature class (dummy: -1)
  L.nb.assign(C, 0);
  for (int p = 0; p < C; ++p) {
    slot_var[p].assign(L.NO, -1);
    slot_class[p].assign(L.NO, -1);
  }
  {
    std::vector<std::vector<int>> mine(C);
    for (int v = 0; v < n_vars; ++v) mine[owner[v]].push_back(v);
    for (int p = 0; p < C; ++p) {
      if (static_cast<int>(mine[p].size()) > L.NO) {
        L.error = "cluster engine: own slots overflow";
        return L;
      }
      std::stable_sort(mine[p].begin(), mine[p].end(), [&](int a, int b) { return sig[a] < sig[b]; });
      for (size_t i = 0; i < mine[p].size(); ++i) {
        slot_var[p][i] = mine[p][i];
        slot_class[p][i] = sig[mine[p][i]];
        L.nb[p] += boundary[mine[p][i]] ? 1 : 0;
      }
    }
    for (int v = 0; v < n_vars; ++v)
      for (int r = 0; r < C; ++r)
        if (r != owner[v] && cnt[static_cast<size_t>(v) * C + r] > 0) ghosts_of[r * C + owner[v]].push_back(v);
  }
  L.gbase.assign(C * C, 0);
  int npl = 0;
  for (int r = 0; r < C; ++r) {
    int s = L.NO;
    for (int o = 0; o < C; ++o) {
      L.gbase[r * C + o] = s;
      for (int v : ghosts_of[r * C + o]) {
        slot_var[r].push_back(v);
        (void)v;
      }
      s += static_cast<int>(ghosts_of[r * C + o].size());
      L.ghost_total += ghosts_of[r * C + o].size();
    }
    slot_var[r].push_back(-1);  // spare
    npl = std::max(npl, s + 1);
  }
  L.NPL = (npl + 31) / 32 * 32;
  // slot_of[p][v] (only for local variables)
  std::vector<std::vector<int>> slot_of(C, std::vector<int>(n_vars, -1));
  auto refresh_slots = [&]() {
    for (int p = 0; p < C; ++p) {
      std::fill(slot_of[p].begin(), slot_of[p].end(), -1);
      for (int s = 0; s < static_cast<int>(slot_var[p].size()); ++s)
        if (slot_var[p][s] >= 0) slot_of[p][slot_var[p][s]] = s;
    }
  };
  refresh_slots();
  // Edge slots inside checks (mutable by the annealer: same-color swaps).
  std::vector<int> eslot(col.edge_slot.begin(), col.edge_slot.end());  // [c * D + r]
  auto spare = [&](int p) { return static_cast<int>(slot_var[p].size()) - 1; };

  // ---- bank annealing: per part, columns (check warp, slot k) over 32 banks ----
  // lc of check c: its index in pchecks[p]; warp = lc % NT / 32 ... thread t handles lc = t + q NT
  std::vector<int> lc_of(M);
  for (int p = 0; p < C; ++p)
    for (int i = 0; i < static_cast<int>(pchecks[p].size()); ++i) lc_of[pchecks[p][i]] = i;
  const int ncolw = NT / 32 * CPT * D;  // columns per part
  std::vector<int> h(static_cast<size_t>(C) * ncolw * 32, 0);
  auto colidx = [&](int c, int k) {
    const int lc = lc_of[c], q = lc / NT, w = (lc % NT) / 32;
    return ((static_cast<size_t>(pc[c]) * ncolw) + (static_cast<size_t>(q) * (NT / 32) + w) * D + k) * 32;
  };
  std::vector<std::vector<int>> var_edges(n_vars);
  for (int c = 0; c < M; ++c)
    for (int r = 0; r < D; ++r) var_edges[rows[c][r]].push_back(c * D + r);
  for (int c = 0; c < M; ++c)
    for (int r = 0; r < D; ++r) h[colidx(c, eslot[c * D + r]) + (slot_of[pc[c]][rows[c][r]] & 31)]++;
  auto total = [&]() {
    double t = 0;
    for (int x : h) t += 0.5 * x * (x - 1);
    return t;
  };
  L.bank_cost_before = total();
  {
    std::mt19937_64 rng(seed + 7);
    std::uniform_real_distribution<double> U(0.0, 1.0);
    auto addh = [&](size_t idx, int d, double& delta) {
      delta += d > 0 ? h[idx] : -(h[idx] - 1);
      h[idx] += d;
    };
    // move variable v's edges inside part p from bank b1 to b2
    auto relocate = [&](int p, int v, int from, int to, double& d) {
      for (int e : var_edges[v]) {
        const int c = e / D;
        if (pc[c] != p) continue;
        const size_t base = colidx(c, eslot[e]);
        addh(base + (from & 31), -1, d);
        addh(base + (to & 31), +1, d);
      }
    };
    double T = 1.0;
    const double decay = std::pow(0.02 / T, 1.0 / static_cast<double>(std::max<long long>(1, bank_moves)));
    for (long long it = 0; it < bank_moves; ++it, T *= decay) {
      const int kind = static_cast<int>(rng() % 3);
      double delta = 0;
      if (kind < 2) {
        // swap two slots of one part: two own slots, or two ghosts of one owner group
        const int p = static_cast<int>(rng() % C);
        int s1, s2;
        if (kind == 0) {
          s1 = static_cast<int>(rng() % L.NO);
          s2 = static_cast<int>(rng() % L.NO);
          if (slot_class[p][s1] != slot_class[p][s2]) continue;  // keep the signature classes
        } else {
          const int o = static_cast<int>(rng() % C);
          const int n = static_cast<int>(ghosts_of[p * C + o].size());
          if (o == p || n < 2) continue;
          s1 = L.gbase[p * C + o] + static_cast<int>(rng() % n);
          s2 = L.gbase[p * C + o] + static_cast<int>(rng() % n);
        }
        if ((s1 & 31) == (s2 & 31)) continue;
        const int v1 = slot_var[p][s1], v2 = slot_var[p][s2];
        if (v1 >= 0) relocate(p, v1, s1, s2, delta);
        if (v2 >= 0) relocate(p, v2, s2, s1, delta);
        if (delta <= 0 || U(rng) < std::exp(-delta / T)) {
          slot_var[p][s1] = v2;
          slot_var[p][s2] = v1;
          if (v1 >= 0) slot_of[p][v1] = s2;
          if (v2 >= 0) slot_of[p][v2] = s1;
        } else {
          double z = 0;
          if (v1 >= 0) relocate(p, v1, s2, s1, z);
          if (v2 >= 0) relocate(p, v2, s1, s2, z);
        }
      } else {
        // swap two same-color slots of one check
        const int c = static_cast<int>(rng() % M);
        const int r1 = static_cast<int>(rng() % D), r2 = static_cast<int>(rng() % D);
        const int e1 = c * D + r1, e2 = c * D + r2;
        const int k1 = eslot[e1], k2 = eslot[e2];
        if (r1 == r2 || k1 % DV != k2 % DV) continue;
        const int p = pc[c];
        const int b1 = slot_of[p][rows[c][r1]] & 31, b2 = slot_of[p][rows[c][r2]] & 31;
        auto apply = [&](int ka, int kb, double& d) {
          addh(colidx(c, ka) + b1, -1, d);
          addh(colidx(c, kb) + b2, -1, d);
          addh(colidx(c, kb) + b1, +1, d);
          addh(colidx(c, ka) + b2, +1, d);
        };
        apply(k1, k2, delta);
        if (delta <= 0 || U(rng) < std::exp(-delta / T)) {
          eslot[e1] = k2;
          eslot[e2] = k1;
        } else {
          double z = 0;
          apply(k2, k1, z);
        }
      }
    }
  }
  L.bank_cost_after = total();

  // ---- device tables ----
  L.chk_slot.assign(static_cast<size_t>(C) * D * L.MC, 0);
  L.chk_orig.assign(static_cast<size_t>(C) * L.MC, -1);
  L.own_var.assign(static_cast<size_t>(C) * L.NO, -1);
  for (int p = 0; p < C; ++p) {
    for (int lc = 0; lc < L.MC; ++lc) {
      const bool act = lc < static_cast<int>(pchecks[p].size());
      const int c = act ? pchecks[p][lc] : -1;
      L.chk_orig[static_cast<size_t>(p) * L.MC + lc] = c;
      for (int k = 0; k < D; ++k) L.chk_slot[(static_cast<size_t>(p) * D + k) * L.MC + lc] = spare(p);
      if (act)
        for (int r = 0; r < D; ++r)
          L.chk_slot[(static_cast<size_t>(p) * D + eslot[c * D + r]) * L.MC + lc] = slot_of[p][rows[c][r]];
    }
    for (int s = 0; s < L.NO; ++s) L.own_var[static_cast<size_t>(p) * L.NO + s] = slot_var[p][s];
  }
  // xsend: part o ships x of its own slot(v) to ghost slot gbase[r][o] + i of part r
  std::vector<std::vector<uint16_t>> xs(C);
  std::vector<std::vector<uint32_t>> ms(C);
  L.xs_start.assign(C * (C + 1), 0);
  L.n_ms.assign(C, 0);
  for (int o = 0; o < C; ++o)
    for (int r = 0; r < C; ++r) {
      L.xs_start[o * (C + 1) + r] = static_cast<int>(xs[o].size());
      if (r == o) continue;
      const int g0 = L.gbase[r * C + o], n = static_cast<int>(ghosts_of[r * C + o].size());
      for (int i = 0; i < n; ++i) xs[o].push_back(static_cast<uint16_t>(slot_of[o][slot_var[r][g0 + i]]));
    }
  for (int o = 0; o < C; ++o) L.xs_start[o * (C + 1) + C] = static_cast<int>(xs[o].size());
  // messages: part p ships the message of its edge (c, v), v owned by o != p,
  // color j, from MSG[j][ghost slot of v here] to MSG[j][own slot of v] of o;
  // sorted by destination word so warps store runs of consecutive words
  struct Msg {
    int o, j, os, gs;
  };
  std::vector<std::vector<Msg>> out(C);
  for (int c = 0; c < M; ++c)
    for (int r = 0; r < D; ++r) {
      const int v = rows[c][r], o = owner[v], p = pc[c];
      if (o == p) continue;
      out[p].push_back({o, eslot[c * D + r] % DV, slot_of[o][v], slot_of[p][v]});
    }
  for (int p = 0; p < C; ++p) {
    std::sort(out[p].begin(), out[p].end(), [](const Msg& a, const Msg& b) {
      return a.o != b.o ? a.o < b.o : a.j != b.j ? a.j < b.j : a.os < b.os;
    });
    for (size_t i = 0; i < out[p].size(); ++i) {
      const Msg& m = out[p][i];
      ms[p].push_back(ms_entry(m.j, m.gs, m.os, m.o));
      if (i == 0 || m.o != out[p][i - 1].o || m.j != out[p][i - 1].j || m.os != out[p][i - 1].os + 1) L.msg_runs++;
    }
    L.n_ms[p] = static_cast<int>(ms[p].size());
    L.msg_total += ms[p].size();
  }
  if (L.NO > 4096 || L.NPL > 8192 || DV > 4) {  // fields of ms_entry / xs_pack
    L.error = "cluster engine: slot space exceeds the packed table fields";
    return L;
  }
  auto cap = [&](size_t m) { return static_cast<int>((m + 31) / 32 * 32); };
  size_t mx = 0, mm = 0;
  for (int p = 0; p < C; ++p) {
    mx = std::max(mx, xs[p].size());
    mm = std::max(mm, ms[p].size());
  }
  L.NXS = cap(mx), L.NMS = cap(mm);
  L.xsend.assign(static_cast<size_t>(C) * L.NXS, 0);
  L.msend.assign(static_cast<size_t>(C) * L.NMS, 0);
  for (int p = 0; p < C; ++p) {
    std::copy(xs[p].begin(), xs[p].end(), L.xsend.begin() + static_cast<size_t>(p) * L.NXS);
    std::copy(ms[p].begin(), ms[p].end(), L.msend.begin() + static_cast<size_t>(p) * L.NMS);
  }
  L.ok = true;
  return L;
}

}  // namespace admm
