// Test harness (CPU): runs the host-side layout builders of csrc/layout.h on
// a code given as flat check lists and reports the layout, so the Python
// tests can verify its invariants without a GPU.
#include <cstdint>
#include <vector>

#include "../../paper_1204_0556_b200/csrc/layout.h"

extern "C" int layout_colored(int n_vars, int n_checks, const int* check_ptr, const int* edge_var, int D, int DV,
                              long long moves, uint64_t seed, int* edge_slot, int* check_rot, int* slot_of_var,
                              double* costs) {
  std::vector<std::vector<int>> rows(n_checks);
  for (int c = 0; c < n_checks; ++c)
    for (int e = check_ptr[c]; e < check_ptr[c + 1]; ++e) rows[c].push_back(edge_var[e]);
  const admm::Layout L = admm::optimize_colored_layout(rows, n_vars, D, DV, moves, seed);
  if (L.clashes) return 1;
  for (int e = 0; e < n_checks * D; ++e) edge_slot[e] = L.edge_slot[e];
  for (int c = 0; c < n_checks; ++c) check_rot[c] = L.check_rot[c];
  for (int v = 0; v < n_vars; ++v) slot_of_var[v] = L.slot_of_var[v];
  costs[0] = L.cost_before;
  costs[1] = L.cost_after;
  return 0;
}

extern "C" int layout_slots(int n_vars, int n_checks, const int* check_ptr, const int* edge_var, int D,
                            long long moves, uint64_t seed, int* edge_slot, int* slot_of_var, double* costs) {
  std::vector<std::vector<int>> rows(n_checks);
  for (int c = 0; c < n_checks; ++c)
    for (int e = check_ptr[c]; e < check_ptr[c + 1]; ++e) rows[c].push_back(edge_var[e]);
  const admm::Layout L = admm::optimize_layout(rows, n_vars, D, moves, seed);
  for (int e = 0; e < n_checks * D; ++e) edge_slot[e] = L.edge_slot[e];
  for (int v = 0; v < n_vars; ++v) slot_of_var[v] = L.slot_of_var[v];
  costs[0] = L.cost_before;
  costs[1] = L.cost_after;
  return L.clashes;
}
