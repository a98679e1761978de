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

template <typename T, int D, int DV, int CPT, int VPT, int MINB, int MAXT, bool COL, int NPC = 0, int NTC = 0,
          bool ZS = false>
ResidentLaunch make_regular() {
  return ResidentLaunch{
      reinterpret_cast<const void*>(&resident_regular_kernel<T, D, DV, CPT, VPT, MINB, MAXT, COL, NPC, NTC, ZS>),
      &launch_regular<T, D, DV, CPT, VPT, MINB, MAXT, COL, NPC, NTC, ZS>, 0, 0, 0, COL, NPC,
      regular_gm_smem(COL, MINB, ZS), ZS ? CPT : 0};
}

// The compiled regular shapes (D, DV, CPT, VPT, MINB, MAXT, COL), in
// preference order.  `variant` selects the variant-th shape that matches
// (D, DV, CPT) and provides at least VPT_min variables per thread; the host
// tries them in turn until one fits the CTA size, registers and shared memory.
//   * fp32 (3,6): colored message layout first (layout.h; no per-edge
//     addresses, no activity predicates in the loop: +10 % on config 2),
//     256-thread CTAs at 3 CTAs/SM (4 CTAs/SM = 64 registers spills: -8 %),
//     then a 704-thread variant for codes with up to 1408
//     checks (config 3);
//   * shared-memory edge state (ZS) only where registers cap the CTAs per SM
//     (config 3: 2 x 448 threads); on config 2 it measured slower at both 5
//     CTAs/SM (712 G) and one check per thread (602 G) than 4 CTAs/SM with
//     the state in registers (836 G);
//   * the slot layout (per-edge message addresses) for everything else and
//     for fp64, whose variable sums must follow the reference's edge order.
template <typename T>
bool regular_lookup_t(int D, int DV, int CPT, int VPT_min, int nt, int n_vars, int variant, int* VPT,
                      ResidentLaunch* out) {
  constexpr bool F32 = sizeof(T) == 4;
  int seen = 0;
#define ADMM_REG(d, dv, cpt, vpt, minb, maxt, col)                               \
  if (D == d && DV == dv && CPT == cpt && VPT_min <= vpt && seen++ == variant) { \
    *VPT = vpt;                                                                  \
    *out = make_regular<T, d, dv, cpt, vpt, minb, maxt, col>();                  \
    return true;                                                                 \
  }
  // compile-time geometry: exactly nt threads and at most npc padded variables
#define ADMM_REG_FIXED(d, dv, cpt, vpt, minb, npc, ntc)                                       \
  if (D == d && DV == dv && CPT == cpt && VPT_min <= vpt && nt == ntc &&                      \
      regular_np(n_vars, true, ntc, vpt) <= npc && seen++ == variant) {                       \
    *VPT = vpt;                                                                               \
    *out = make_regular<T, d, dv, cpt, vpt, minb, ntc, true, npc, ntc>();                     \
    return true;                                                                              \
  }
  // ... with the edge state in shared memory (ZS)
#define ADMM_REG_FIXED_ZS(d, dv, cpt, vpt, minb, npc, ntc)                                    \
  if (D == d && DV == dv && CPT == cpt && VPT_min <= vpt && nt == ntc &&                      \
      regular_np(n_vars, true, ntc, vpt) <= npc && seen++ == variant) {                       \
    *VPT = vpt;                                                                               \
    *out = make_regular<T, d, dv, cpt, vpt, minb, ntc, true, npc, ntc, true>();               \
    return true;                                                                              \
  }
  if constexpr (F32) {
    ADMM_REG_FIXED_ZS(6, 3, 3, 6, 2, 2688, 448)
    ADMM_REG_FIXED(6, 3, 2, 4, 4, 1024, 256)
    ADMM_REG_FIXED(6, 3, 2, 4, 3, 1024, 256)
    ADMM_REG_FIXED(6, 3, 2, 4, 1, 2688, 672)
    ADMM_REG_FIXED(13, 3, 1, 6, 2, 1536, 256)
    ADMM_REG(6, 3, 2, 4, 3, 256, true)
    ADMM_REG(6, 3, 2, 4, 1, 704, true)
    ADMM_REG(6, 3, 1, 2, 2, 512, true)
  }
  if constexpr (!F32) {  // fp64: colored layout with compile-time geometry (color-order variable sums)
    ADMM_REG_FIXED(6, 3, 2, 4, 2, 1024, 256)
  }
  ADMM_REG(6, 3, 1, 2, F32 ? 2 : 1, 512, false)
  ADMM_REG(6, 3, 2, 4, F32 ? 3 : 1, F32 ? 256 : 512, false)
  ADMM_REG(6, 3, 2, 4, 1, 704, false)
  ADMM_REG(6, 3, 3, 6, 1, 512, false)
  ADMM_REG(6, 3, 4, 8, 1, 512, false)
  ADMM_REG(13, 3, 1, 5, 1, 512, false)
  ADMM_REG(4, 2, 1, 2, F32 ? 2 : 1, 512, false)
  ADMM_REG(4, 3, 1, 2, F32 ? 2 : 1, 512, false)
#undef ADMM_REG
#undef ADMM_REG_FIXED
#undef ADMM_REG_FIXED_ZS
  return false;
}

}  // namespace admm
