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

template <typename T, int D, int DV, int CPT, int VPT>
ResidentLaunch make_regular() {
  // CPT = 2, d <= 8, fp32: a 256-thread CTA bounded to 85 registers so three
  // CTAs fit an SM (ADMM_B200_MINB3 selects it for A/B measurements).
  constexpr bool k3 = sizeof(T) == 4 && CPT == 2 && D <= 8;
  constexpr int MINB = (sizeof(T) == 4 && CPT == 1 && D <= 8) ? 2 : k3 ? 3 : 1;
  constexpr int MAXT = k3 ? 256 : 512;
  return ResidentLaunch{reinterpret_cast<const void*>(&resident_regular_kernel<T, D, DV, CPT, VPT, MINB, MAXT>),
                        &launch_regular<T, D, DV, CPT, VPT, MINB, MAXT>, 0, 0, 0};
}

// The compiled regular shapes.  VPT is the smallest compiled value >= the
// variables-per-thread the graph needs.
template <typename T>
bool regular_lookup_t(int D, int DV, int CPT, int VPT_min, int* VPT, ResidentLaunch* out) {
#define ADMM_REG(d, dv, cpt, vpt)                                         \
  if (D == d && DV == dv && CPT == cpt && VPT_min <= vpt) {               \
    *VPT = vpt;                                                           \
    *out = make_regular<T, d, dv, cpt, vpt>();                            \
    return true;                                                          \
  }
  ADMM_REG(6, 3, 1, 2)
  ADMM_REG(6, 3, 2, 4)
  ADMM_REG(6, 3, 3, 6)
  ADMM_REG(6, 3, 4, 8)
  ADMM_REG(13, 3, 1, 5)
  ADMM_REG(4, 2, 1, 2)
  ADMM_REG(4, 3, 1, 2)
#undef ADMM_REG
  return false;
}

}  // namespace admm
