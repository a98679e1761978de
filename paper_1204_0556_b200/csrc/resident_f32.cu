#include "resident_inst.cuh"
namespace admm {
bool resident_lookup_f32(int D, int CPT, int DVMAX, ResidentLaunch* out) {
  return resident_lookup_t<float>(D, CPT, DVMAX, out);
}
}  // namespace admm
