#include "resident_inst.cuh"
namespace admm {
bool resident_lookup_f32(int D, int CPT, int DVMAX, ResidentLaunch* out) {
  return resident_lookup_t<float>(D, CPT, DVMAX, out);
}
bool regular_lookup_f32(int D, int DV, int CPT, int VPT_min, int nt, int n_vars, int variant, int* VPT,
                        ResidentLaunch* out) {
  return regular_lookup_t<float>(D, DV, CPT, VPT_min, nt, n_vars, variant, VPT, out);
}
}  // namespace admm
