// Bank-conflict-aware relabeling of the Tanner graph for the regular
// resident kernel (host code, run once in admm_graph_create).
//
// The kernel's shared-memory gathers are:
//   x-gather   warp = 32 consecutive (internal) checks, slot k:   address x[pi(v)]
//   msg-gather warp = 32 consecutive (internal) variables, edge j: address msg[c*DS + k(c,v)]
// (fp32: bank = word address mod 32).  Both the internal variable numbering
// pi and the slot k of every edge inside its check are free: the projection
// is permutation-equivariant and a variable still sums its messages in
// increasing check order, so results are unchanged.  This module searches
// (pi, k) by simulated annealing to minimise sum over gather groups of
// sum_bank count^2 -- 32 lanes on 32 distinct banks is one wavefront.
#pragma once

#include <cmath>
#include <cstdint>
#include <algorithm>
#include <random>
#include <vector>

namespace admm {

struct Layout {
  std::vector<int> var_of_slot;   // internal var index -> original var
  std::vector<int> slot_of_var;   // original var -> internal var index
  std::vector<int> edge_slot;     // per original edge (check-major, sorted rows): slot k inside its check
  double cost_before = 0, cost_after = 0;
};

// rows[c] = sorted original variables of check c (all of size D); each
// variable has degree DV.  ds = message row stride (odd).
inline Layout optimize_layout(const std::vector<std::vector<int>>& rows, int n_vars, int D, int DV, int ds,
                              long long moves, uint64_t seed) {
  const int M = static_cast<int>(rows.size());
  Layout L;
  std::mt19937_64 rng(seed);
  // edges: e = c*D + (index in sorted row)
  std::vector<int> ev(static_cast<size_t>(M) * D), ec(static_cast<size_t>(M) * D);
  std::vector<std::vector<int>> var_edges(n_vars);  // increasing check order
  for (int c = 0; c < M; ++c)
    for (int r = 0; r < D; ++r) {
      const int e = c * D + r;
      ev[e] = rows[c][r];
      ec[e] = c;
      var_edges[rows[c][r]].push_back(e);
    }
  std::vector<int> jidx(static_cast<size_t>(M) * D);  // position of edge e in its variable's edge list
  for (int v = 0; v < n_vars; ++v)
    for (size_t j = 0; j < var_edges[v].size(); ++j) jidx[var_edges[v][j]] = static_cast<int>(j);

  L.slot_of_var.resize(n_vars);
  L.var_of_slot.resize(n_vars);
  for (int v = 0; v < n_vars; ++v) L.var_of_slot[v] = v;
  std::shuffle(L.var_of_slot.begin(), L.var_of_slot.end(), rng);
  for (int i = 0; i < n_vars; ++i) L.slot_of_var[L.var_of_slot[i]] = i;
  L.edge_slot.resize(static_cast<size_t>(M) * D);
  std::vector<int> slot_edge(static_cast<size_t>(M) * D);  // (c, k) -> edge
  for (int e = 0; e < M * D; ++e) {
    L.edge_slot[e] = e % D;
    slot_edge[e] = e;
  }

  // Histograms: group A (check-warp, slot) over banks of pi(v);
  //             group B (var-warp, j)     over banks of (ds*c + k).
  const int nA = (M + 31) / 32 * D, nB = (n_vars + 31) / 32 * DV;
  std::vector<int> hA(static_cast<size_t>(nA) * 32, 0), hB(static_cast<size_t>(nB) * 32, 0);
  auto keyA = [&](int c, int k) { return ((c >> 5) * D + k) * 32; };
  auto keyB = [&](int slot, int j) { return ((slot >> 5) * DV + j) * 32; };
  auto bankB = [&](int c, int k) { return (ds * c + k) & 31; };
  for (int e = 0; e < M * D; ++e) {
    const int c = ec[e], v = ev[e], k = L.edge_slot[e];
    hA[keyA(c, k) + (L.slot_of_var[v] & 31)]++;
    hB[keyB(L.slot_of_var[v], jidx[e]) + bankB(c, k)]++;
  }
  auto total = [&]() {
    double s = 0;
    for (int x : hA) s += double(x) * x;
    for (int x : hB) s += double(x) * x;
    return s;
  };
  L.cost_before = total();
  // Changing one histogram entry by +-1 changes sum(count^2) by 2*count+1 / -2*count+1.
  auto add = [](std::vector<int>& h, int idx, int d, double& delta) {
    delta += d > 0 ? 2.0 * h[idx] + 1 : -2.0 * h[idx] + 1;
    h[idx] += d;
  };
  std::uniform_real_distribution<double> U(0.0, 1.0);
  double T = 2.0;
  const double T_end = 0.02;
  const double decay = std::pow(T_end / T, 1.0 / std::max<long long>(1, moves));
  for (long long it = 0; it < moves; ++it, T *= decay) {
    double delta = 0;
    if (U(rng) < 0.5) {
      // swap internal slots of two variables
      const int v1 = static_cast<int>(rng() % n_vars), v2 = static_cast<int>(rng() % n_vars);
      if (v1 == v2) continue;
      const int s1 = L.slot_of_var[v1], s2 = L.slot_of_var[v2];
      auto relocate = [&](int v, int from, int to, double& d) {
        for (int e : var_edges[v]) {
          const int c = ec[e], k = L.edge_slot[e];
          add(hA, keyA(c, k) + (from & 31), -1, d);
          add(hA, keyA(c, k) + (to & 31), +1, d);
          add(hB, keyB(from, jidx[e]) + bankB(c, k), -1, d);
          add(hB, keyB(to, jidx[e]) + bankB(c, k), +1, d);
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
      const int b1 = L.slot_of_var[ev[e1]], b2 = L.slot_of_var[ev[e2]];
      auto place = [&](int e, int slot_v, int k, int sign) {
        add(hA, keyA(c, k) + (slot_v & 31), sign, delta);
        add(hB, keyB(slot_v, jidx[e]) + bankB(c, k), sign, delta);
      };
      place(e1, b1, k1, -1);
      place(e2, b2, k2, -1);
      place(e1, b1, k2, +1);
      place(e2, b2, k1, +1);
      if (delta <= 0 || U(rng) < std::exp(-delta / T)) {
        L.edge_slot[e1] = k2;
        L.edge_slot[e2] = k1;
        slot_edge[c * D + k2] = e1;
        slot_edge[c * D + k1] = e2;
      } else {
        double z = 0;
        auto undo = [&](int e, int slot_v, int k, int sign) {
          add(hA, keyA(c, k) + (slot_v & 31), sign, z);
          add(hB, keyB(slot_v, jidx[e]) + bankB(c, k), sign, z);
        };
        undo(e1, b1, k2, -1);
        undo(e2, b2, k1, -1);
        undo(e1, b1, k1, +1);
        undo(e2, b2, k2, +1);
      }
    }
  }
  L.cost_after = total();
  return L;
}

}  // namespace admm
