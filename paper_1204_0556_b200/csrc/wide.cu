// Instantiations of the wide streaming engine (wide.cuh): dtype x check-degree
// bucket x variable-degree bucket, with the regular (fixed-degree projection)
// variants for the BASELINE degrees.  VS (slots per thread) shrinks with the
// check degree so the D x VS x 3 loaded words stay in registers.
#include <cstdlib>

#include "kernels.cuh"

namespace admm {

template <typename T, int VS, int D, int DV, bool REG, int NS = 2, int MINB = 2>
WideLaunch wide_entry() {
  return WideLaunch{reinterpret_cast<const void*>(&wide_decode_kernel<T, VS, D, DV, REG, NS, MINB>),
                    &launch_wide<T, VS, D, DV, REG, NS, MINB>, 0, 0, VS, wide_smem_bytes<T, VS, D, DV, NS>(), D, DV};
}

template <typename T, int DV>
bool wide_lookup_dv(int D, bool regular, WideLaunch* out) {
  constexpr int VS = sizeof(T) == 4 ? 2 : 1;  // z/lambda of a thread's slots: one 16-byte access
  if constexpr (DV == 3) {
    if (!regular) return false;
    switch (D) {
      case 6: *out = wide_entry<T, VS, 6, 3, true>(); return true;
      case 13: *out = wide_entry<T, 1, 13, 3, true>(); return true;
      default: return false;
    }
  } else {
    switch (D) {
      case 4: *out = wide_entry<T, VS, 4, DV, false>(); return true;
      case 6: *out = wide_entry<T, VS, 6, DV, false>(); return true;
      case 8: *out = wide_entry<T, VS, 8, DV, false>(); return true;
      default: return false;
    }
  }
}

bool wide_lookup(int dtype, int D, int DVMAX, bool regular, WideLaunch* out) {
  if (regular && DVMAX == 3)
    return dtype ? wide_lookup_dv<double, 3>(D, true, out) : wide_lookup_dv<float, 3>(D, true, out);
  if (DVMAX <= 4) return dtype ? wide_lookup_dv<double, 4>(D, false, out) : wide_lookup_dv<float, 4>(D, false, out);
  return false;
}

bool wide_phase_profile(int enable, unsigned long long* out8) {
  if (out8) {
    if (cudaMemcpyFromSymbol(out8, g_wide_cycles, sizeof(unsigned long long) * 8) != cudaSuccess) return false;
  }
  if (enable >= 0) {
    const unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const int on = enable > 0;
    if (cudaMemcpyToSymbol(g_wide_cycles, z, sizeof(z)) != cudaSuccess) return false;
    if (cudaMemcpyToSymbol(g_wide_prof, &on, sizeof(int)) != cudaSuccess) return false;
  }
  return true;
}

}  // namespace admm
