// Bank-conflict-free layout of the Tanner graph for the regular resident
// kernel (host code, run once in admm_graph_create).
//
// Shared-memory layout of the kernel (fp32 bank = word address mod 32):
//     x   [Npad]            x of internal variable i at word i
//     msg [D][Npad]         message of edge (c, v) at word k*Npad + pi(v),
//                           k = the edge's slot inside check c
// with Npad a multiple of 32.  The accesses are:
//   var phase   a warp = 32 consecutive internal variables i; loads
//               msg[k_j(i)][i] for j < DV and stores x[i]: bank = i mod 32,
//               conflict-free BY CONSTRUCTION;
//   check phase a warp = 32 consecutive checks; for slot k it loads x[pi(v)]
//               and stores msg[k][pi(v)]: bank = pi(v) mod 32 for both.
// So one constraint family remains: inside every (check-warp, slot k) column
// the 32 variables must have distinct pi(v) mod 32.  The message buffer
// additionally needs the DV edges of a variable in DISTINCT slots (they share
// the word msg[k][pi(v)] otherwise).  Both the internal numbering pi and the
// slot of every edge inside its check are free -- the projection is
// permutation-equivariant and a variable still sums its messages in
// increasing check order -- so results are unchanged.  Simulated annealing
// over (pi swaps, in-check slot swaps) minimises
//     sum over columns of sum_bank C(count, 2)  +  W * (slot clashes)
// and reports the resulting wavefront histogram.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <random>
#include <vector>

namespace admm {

struct Layout {
  std::vector<int> var_of_slot;  // internal var index -> original var
  std::vector<int> slot_of_var;  // original var -> internal var index
  std::vector<int> edge_slot;    // per original edge (c*D + sorted position): slot k inside check c
  std::vector<int> check_rot;    // colored layout: rotation r_c (slot k has color (k + r_c) mod DV)
  double cost_before = 0, cost_after = 0;
  int clashes = 0;               // variables with two edges in one slot (must be 0 to use the layout)
  int max_wavefronts = 0;        // worst column after optimisation
};

inline Layout optimize_layout(const std::vector<std::vector<int>>& rows, int n_vars, int D, long long moves,
                              uint64_t seed) {
  const int M = static_cast<int>(rows.size());
  const int E = M * D;
  Layout L;
  std::mt19937_64 rng(seed);
  std::vector<int> ev(E), ec(E);
  std::vector<std::vector<int>> var_edges(n_vars);
  for (int c = 0; c < M; ++c)
    for (int r = 0; r < D; ++r) {
      ev[c * D + r] = rows[c][r];
      ec[c * D + r] = c;
      var_edges[rows[c][r]].push_back(c * D + r);
    }
  L.slot_of_var.resize(n_vars);
  L.var_of_slot.resize(n_vars);
  for (int v = 0; v < n_vars; ++v) L.var_of_slot[v] = v;
  std::shuffle(L.var_of_slot.begin(), L.var_of_slot.end(), rng);
  for (int i = 0; i < n_vars; ++i) L.slot_of_var[L.var_of_slot[i]] = i;
  L.edge_slot.resize(E);
  std::vector<int> slot_edge(E);
  for (int e = 0; e < E; ++e) {
    L.edge_slot[e] = e % D;
    slot_edge[e] = e;
  }
  // Column histograms (check-warp, k) over banks, and per-variable slot use.
  const int ncol = (M + 31) / 32 * D;
  std::vector<int> h(static_cast<size_t>(ncol) * 32, 0), vs(static_cast<size_t>(n_vars) * D, 0);
  auto col = [&](int c, int k) { return ((c >> 5) * D + k) * 32; };
  for (int e = 0; e < E; ++e) {
    h[col(ec[e], L.edge_slot[e]) + (L.slot_of_var[ev[e]] & 31)]++;
    vs[static_cast<size_t>(ev[e]) * D + L.edge_slot[e]]++;
  }
  const double W = 4.0;
  auto total = [&]() {
    double s = 0;
    for (int x : h) s += 0.5 * x * (x - 1);
    for (int x : vs) s += W * 0.5 * x * (x - 1);
    return s;
  };
  // +-1 on a count x changes C(x,2) by +x / -(x-1).
  auto addh = [&](int idx, int d, double& delta) {
    delta += d > 0 ? h[idx] : -(h[idx] - 1);
    h[idx] += d;
  };
  auto addv = [&](size_t idx, int d, double& delta) {
    delta += W * (d > 0 ? vs[idx] : -(vs[idx] - 1));
    vs[idx] += d;
  };
  L.cost_before = total();
  std::uniform_real_distribution<double> U(0.0, 1.0);
  double T = 1.0;
  const double decay = std::pow(0.02 / T, 1.0 / static_cast<double>(std::max<long long>(1, moves)));
  for (long long it = 0; it < moves; ++it, T *= decay) {
    double delta = 0;
    if (rng() & 1) {
      // swap the internal indices of two variables (moves their banks)
      const int v1 = static_cast<int>(rng() % n_vars), v2 = static_cast<int>(rng() % n_vars);
      if (v1 == v2) continue;
      const int s1 = L.slot_of_var[v1], s2 = L.slot_of_var[v2];
      if ((s1 & 31) == (s2 & 31)) continue;
      auto relocate = [&](int v, int from, int to, double& d) {
        for (int e : var_edges[v]) {
          const int base = col(ec[e], L.edge_slot[e]);
          addh(base + (from & 31), -1, d);
          addh(base + (to & 31), +1, d);
        }
      };
      relocate(v1, s1, s2, delta);
      relocate(v2, s2, s1, delta);
      if (delta <= 0 || U(rng) < std::exp(-delta / T)) {
        L.slot_of_var[v1] = s2;
        L.slot_of_var[v2] = s1;
        L.var_of_slot[s2] = v1;
        L.var_of_slot[s1] = v2;
      } else {
        double z = 0;
        relocate(v1, s2, s1, z);
        relocate(v2, s1, s2, z);
      }
    } else {
      // swap the slots of two edges of one check
      const int c = static_cast<int>(rng() % M);
      const int k1 = static_cast<int>(rng() % D), k2 = static_cast<int>(rng() % D);
      if (k1 == k2) continue;
      const int e1 = slot_edge[c * D + k1], e2 = slot_edge[c * D + k2];
      const int b1 = L.slot_of_var[ev[e1]] & 31, b2 = L.slot_of_var[ev[e2]] & 31;
      const size_t v1 = static_cast<size_t>(ev[e1]) * D, v2 = static_cast<size_t>(ev[e2]) * D;
      auto apply = [&](int ka, int kb, double& d) {  // e1: ka -> kb, e2: kb -> ka
        addh(col(c, ka) + b1, -1, d);
        addh(col(c, kb) + b2, -1, d);
        addh(col(c, kb) + b1, +1, d);
        addh(col(c, ka) + b2, +1, d);
        addv(v1 + ka, -1, d);
        addv(v2 + kb, -1, d);
        addv(v1 + kb, +1, d);
        addv(v2 + ka, +1, d);
      };
      apply(k1, k2, delta);
      if (delta <= 0 || U(rng) < std::exp(-delta / T)) {
        L.edge_slot[e1] = k2;
        L.edge_slot[e2] = k1;
        slot_edge[c * D + k2] = e1;
        slot_edge[c * D + k1] = e2;
      } else {
        double z = 0;
        apply(k2, k1, z);
      }
    }
  }
  L.cost_after = total();
  L.clashes = 0;
  for (int x : vs) L.clashes += x > 1;
  L.max_wavefronts = 0;
  for (int x : h) L.max_wavefronts = std::max(L.max_wavefronts, x);
  return L;
}


// Colored layout for regular codes with D = q DV + rem, rem in {0, 1} (the
// (3,6) and (3,13) codes): every edge gets a color j in [0, DV) such that
// each variable has one edge of every color and each check q edges of every
// color plus, when rem = 1, one more edge of its ROTATION color r_c; the
// check's color-j edges sit in the slots k with (k + r_c) mod DV = j.  The
// message of edge (c, v) of color j is stored at msgc[j][pi(v)]: a variable
// reads its messages at compile-time offsets from its own x slot and a check
// writes slot k at offset (k + r_c) mod DV from the address it gathered x
// from -- no per-edge message addresses anywhere.
//
// Existence (Koenig): split every check into q copies of degree DV and, when
// rem = 1, one copy of degree 1 padded with DV - 1 edges to M (DV - 1) / DV
// dummy variables of degree DV.  The result is a DV-regular bipartite
// multigraph, i.e. the union of DV perfect matchings; color j = matching j,
// and r_c = the color of the check's degree-1 copy.  The annealer then moves
// variables (pi) and swaps same-color slots of one check to spread every
// (check-warp, slot) column over the 32 banks.
inline bool match_dfs(int v, const std::vector<std::vector<int>>& adj, const std::vector<char>& used_edge,
                      const std::vector<int>& edge_copy, std::vector<int>& copy_match, std::vector<int>& seen,
                      int stamp, std::vector<int>& var_match_edge) {
  for (int e : adj[v]) {
    if (used_edge[e]) continue;
    const int cp = edge_copy[e];
    if (seen[cp] == stamp) continue;
    seen[cp] = stamp;
    if (copy_match[cp] < 0 ||
        match_dfs(copy_match[cp], adj, used_edge, edge_copy, copy_match, seen, stamp, var_match_edge)) {
      copy_match[cp] = v;
      var_match_edge[v] = e;
      return true;
    }
  }
  return false;
}

inline bool colored_layout_supported(int M, int D, int DV) {
  const int rem = D % DV;
  return DV >= 1 && D >= DV && (rem == 0 || (rem == 1 && (M * (DV - 1)) % DV == 0));
}

inline Layout optimize_colored_layout(const std::vector<std::vector<int>>& rows, int n_vars, int D, int DV,
                                      long long moves, uint64_t seed) {
  const int M = static_cast<int>(rows.size());
  const int E = M * D, Q = D / DV, rem = D % DV;
  Layout L;
  if (!colored_layout_supported(M, D, DV)) {
    L.clashes = 1;
    return L;
  }
  std::mt19937_64 rng(seed);
  const int CPC = Q + (rem ? 1 : 0);           // copies per check
  const int NCOPY = M * CPC;
  const int ND = rem ? M * (DV - 1) / DV : 0;  // dummy variables
  const int ED = rem ? M * (DV - 1) : 0;       // dummy edges
  std::vector<int> ev(E + ED), ec(E), edge_copy(E + ED), color(E + ED, -1);
  std::vector<std::vector<int>> adj(n_vars + ND);
  for (int c = 0; c < M; ++c) {
    std::vector<int> perm(D);
    for (int r = 0; r < D; ++r) perm[r] = r;
    std::shuffle(perm.begin(), perm.end(), rng);
    for (int r = 0; r < D; ++r) {
      const int e = c * D + r;
      ev[e] = rows[c][r];
      ec[e] = c;
      edge_copy[e] = c * CPC + perm[r] / DV;  // perm == D - 1 (rem = 1) -> the degree-1 copy
      adj[ev[e]].push_back(e);
    }
  }
  for (int t = 0; t < ED; ++t) {  // pad every degree-1 copy with DV - 1 dummy edges
    const int c = t / (DV - 1), e = E + t, d = n_vars + t / DV;
    ev[e] = d;
    edge_copy[e] = c * CPC + Q;
    adj[d].push_back(e);
  }
  // DV successive perfect matchings of the DV-regular multigraph.
  const int NL = n_vars + ND;
  std::vector<char> used(E + ED, 0);
  std::vector<int> seen(NCOPY, -1);
  int stamp = 0;
  for (int j = 0; j < DV; ++j) {
    std::vector<int> copy_match(NCOPY, -1), var_edge(NL, -1);
    for (int v = 0; v < NL; ++v) {
      if (!match_dfs(v, adj, used, edge_copy, copy_match, seen, stamp++, var_edge)) {
        L.clashes = 1;  // cannot happen for a biregular graph (Koenig)
        return L;
      }
    }
    for (int v = 0; v < NL; ++v) {
      used[var_edge[v]] = 1;
      color[var_edge[v]] = j;
    }
  }
  // Rotations and slots: the color-j edges of check c take the slots k with
  // (k + r_c) mod DV == j, in increasing k.
  L.check_rot.assign(M, 0);
  if (rem)
    for (int e = 0; e < E; ++e)
      if (edge_copy[e] == ec[e] * CPC + Q) L.check_rot[ec[e]] = color[e];
  L.edge_slot.assign(E, -1);
  std::vector<int> slot_edge(E);
  std::vector<std::vector<std::vector<int>>> color_slots(M);  // [c][j] -> slots
  for (int c = 0; c < M; ++c) {
    color_slots[c].assign(DV, {});
    for (int k = 0; k < D; ++k) color_slots[c][(k + L.check_rot[c]) % DV].push_back(k);
    std::vector<int> fill(DV, 0);
    for (int r = 0; r < D; ++r) {
      const int e = c * D + r, j = color[e];
      if (fill[j] >= static_cast<int>(color_slots[c][j].size())) {
        L.clashes = 1;
        return L;
      }
      const int k = color_slots[c][j][fill[j]++];
      L.edge_slot[e] = k;
      slot_edge[c * D + k] = e;
    }
  }
  L.slot_of_var.resize(n_vars);
  L.var_of_slot.resize(n_vars);
  for (int v = 0; v < n_vars; ++v) L.var_of_slot[v] = v;
  std::shuffle(L.var_of_slot.begin(), L.var_of_slot.end(), rng);
  for (int i = 0; i < n_vars; ++i) L.slot_of_var[L.var_of_slot[i]] = i;
  std::vector<std::vector<int>> var_edges(n_vars);
  for (int e = 0; e < E; ++e) var_edges[ev[e]].push_back(e);
  const int ncol = (M + 31) / 32 * D;
  std::vector<int> h(static_cast<size_t>(ncol) * 32, 0);
  auto col = [&](int c, int k) { return ((c >> 5) * D + k) * 32; };
  for (int e = 0; e < E; ++e) h[col(ec[e], L.edge_slot[e]) + (L.slot_of_var[ev[e]] & 31)]++;
  auto total = [&]() {
    double t = 0;
    for (int x : h) t += 0.5 * x * (x - 1);
    return t;
  };
  auto addh = [&](int idx, int d, double& delta) {
    delta += d > 0 ? h[idx] : -(h[idx] - 1);
    h[idx] += d;
  };
  L.cost_before = total();
  std::uniform_real_distribution<double> U(0.0, 1.0);
  double T = 1.0;
  const double decay = std::pow(0.02 / T, 1.0 / static_cast<double>(std::max<long long>(1, moves)));
  for (long long it = 0; it < moves; ++it, T *= decay) {
    double delta = 0;
    if (Q < 2 || (rng() & 1)) {
      const int v1 = static_cast<int>(rng() % n_vars), v2 = static_cast<int>(rng() % n_vars);
      if (v1 == v2) continue;
      const int s1 = L.slot_of_var[v1], s2 = L.slot_of_var[v2];
      if ((s1 & 31) == (s2 & 31)) continue;
      auto relocate = [&](int v, int from, int to, double& d) {
        for (int e : var_edges[v]) {
          const int base = col(ec[e], L.edge_slot[e]);
          addh(base + (from & 31), -1, d);
          addh(base + (to & 31), +1, d);
        }
      };
      relocate(v1, s1, s2, delta);
      relocate(v2, s2, s1, delta);
      if (delta <= 0 || U(rng) < std::exp(-delta / T)) {
        L.slot_of_var[v1] = s2;
        L.slot_of_var[v2] = s1;
        L.var_of_slot[s2] = v1;
        L.var_of_slot[s1] = v2;
      } else {
        double z = 0;
        relocate(v1, s2, s1, z);
        relocate(v2, s1, s2, z);
      }
    } else {
      // swap two same-color slots of one check
      const int c = static_cast<int>(rng() % M);
      const std::vector<int>& cs = color_slots[c][rng() % DV];
      const int a = static_cast<int>(rng() % cs.size()), b = static_cast<int>(rng() % cs.size());
      if (a == b) continue;
      const int k1 = cs[a], k2 = cs[b];
      const int e1 = slot_edge[c * D + k1], e2 = slot_edge[c * D + k2];
      const int b1 = L.slot_of_var[ev[e1]] & 31, b2 = L.slot_of_var[ev[e2]] & 31;
      auto apply = [&](int ka, int kb, double& d) {
        addh(col(c, ka) + b1, -1, d);
        addh(col(c, kb) + b2, -1, d);
        addh(col(c, kb) + b1, +1, d);
        addh(col(c, ka) + b2, +1, d);
      };
      apply(k1, k2, delta);
      if (delta <= 0 || U(rng) < std::exp(-delta / T)) {
        L.edge_slot[e1] = k2;
        L.edge_slot[e2] = k1;
        slot_edge[c * D + k2] = e1;
        slot_edge[c * D + k1] = e2;
      } else {
        double z = 0;
        apply(k2, k1, z);
      }
    }
  }
  L.cost_after = total();
  L.clashes = 0;
  L.max_wavefronts = 0;
  for (int x : h) L.max_wavefronts = std::max(L.max_wavefronts, x);
  return L;
}

}  // namespace admm
