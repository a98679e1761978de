#include "resident_inst.cuh"
namespace admm {
bool resident_lookup_f64(int D, int CPT, int DVMAX, ResidentLaunch* out) {
  return resident_lookup_t<double>(D, CPT, DVMAX, out);
}
}  // namespace admm
