// Instantiation table for one dtype (included by resident_f32.cu / _f64.cu).
#pragma once
#include "kernels.cuh"

namespace admm {

template <typename T, int D, int CPT, int DVMAX>
ResidentLaunch make_entry() {
  return ResidentLaunch{reinterpret_cast<const void*>(&resident_decode_kernel<T, D, CPT, DVMAX>),
                        &launch_resident<T, D, CPT, DVMAX>, 0, 0, 0};
}

template <typename T, int D, int DVMAX>
bool lookup_cpt(int CPT, ResidentLaunch* out) {
  switch (CPT) {
    case 1: *out = make_entry<T, D, 1, DVMAX>(); return true;
    case 2: *out = make_entry<T, D, 2, DVMAX>(); return true;
    case 4: *out = make_entry<T, D, 4, DVMAX>(); return true;
  }
  return false;
}

template <typename T, int D>
bool lookup_dv(int CPT, int DVMAX, ResidentLaunch* out) {
  if (DVMAX == 4) return lookup_cpt<T, D, 4>(CPT, out);
  if (DVMAX == 8) return lookup_cpt<T, D, 8>(CPT, out);
  return false;
}

template <typename T>
bool resident_lookup_t(int D, int CPT, int DVMAX, ResidentLaunch* out) {
  switch (D) {
    case 4: return lookup_dv<T, 4>(CPT, DVMAX, out);
    case 6: return lookup_dv<T, 6>(CPT, DVMAX, out);
    case 8: return lookup_dv<T, 8>(CPT, DVMAX, out);
    case 13: return lookup_dv<T, 13>(CPT, DVMAX, out);
    case 16: return lookup_dv<T, 16>(CPT, DVMAX, out);
    case 32: return CPT == 1 ? lookup_dv<T, 32>(1, DVMAX, out) : false;
  }
  return false;
}

template <typename T, int D, int DV, int CPT, int VPT, int MINB, int MAXT>
ResidentLaunch make_regular() {
  return ResidentLaunch{reinterpret_cast<const void*>(&resident_regular_kernel<T, D, DV, CPT, VPT, MINB, MAXT>),
                        &launch_regular<T, D, DV, CPT, VPT, MINB, MAXT>, 0, 0, 0};
}

// The compiled regular shapes (D, DV, CPT, VPT, MINB, MAXT), in preference
// order.  `variant` selects the variant-th shape that matches (D, DV, CPT)
// and provides at least VPT_min variables per thread; the host tries them in
// turn until one fits the CTA size, registers and shared memory.
//   * fp32, CPT = 2: 256-thread CTAs bounded to 85 registers (3 CTAs/SM,
//     +1.3 % over 2 CTAs on config 2), then a 704-thread variant for codes
//     with up to 1408 checks (config 3: 672 threads, 21 warps).
template <typename T>
bool regular_lookup_t(int D, int DV, int CPT, int VPT_min, int variant, int* VPT, ResidentLaunch* out) {
  constexpr bool F32 = sizeof(T) == 4;
  int seen = 0;
#define ADMM_REG(d, dv, cpt, vpt, minb, maxt)                               \
  if (D == d && DV == dv && CPT == cpt && VPT_min <= vpt && seen++ == variant) { \
    *VPT = vpt;                                                             \
    *out = make_regular<T, d, dv, cpt, vpt, minb, maxt>();                  \
    return true;                                                            \
  }
  ADMM_REG(6, 3, 1, 2, F32 ? 2 : 1, 512)
  ADMM_REG(6, 3, 2, 4, F32 ? 3 : 1, F32 ? 256 : 512)
  ADMM_REG(6, 3, 2, 4, 1, 704)
  ADMM_REG(6, 3, 3, 6, 1, 512)
  ADMM_REG(6, 3, 4, 8, 1, 512)
  ADMM_REG(13, 3, 1, 5, 1, 512)
  ADMM_REG(4, 2, 1, 2, F32 ? 2 : 1, 512)
  ADMM_REG(4, 3, 1, 2, F32 ? 2 : 1, 512)
#undef ADMM_REG
  return false;
}

}  // namespace admm
