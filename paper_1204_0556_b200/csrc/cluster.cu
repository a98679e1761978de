// Instantiations of the cluster-resident engine (regular codes).
#include "kernels.cuh"

namespace admm {

template <typename T, int D, int DV, int CPT, int VPT>
ClusterLaunch cluster_entry() {
  return ClusterLaunch{reinterpret_cast<const void*>(&cluster_decode_kernel<T, D, DV, CPT, VPT>),
                       &launch_cluster<T, D, DV, CPT, VPT>, 0, 0, 0};
}

template <typename T>
bool cluster_lookup_t(int D, int DV, int CPT, int VPT_min, int* VPT, ClusterLaunch* out) {
#define ADMM_CL(d, dv, cpt, vpt)                          \
  if (D == d && DV == dv && CPT == cpt && VPT_min <= vpt) { \
    *VPT = vpt;                                           \
    *out = cluster_entry<T, d, dv, cpt, vpt>();           \
    return true;                                          \
  }
  ADMM_CL(6, 3, 1, 2)
  ADMM_CL(6, 3, 2, 4)
  ADMM_CL(13, 3, 1, 5)
#undef ADMM_CL
  return false;
}

bool cluster_lookup(int dtype, int D, int DV, int CPT, int VPT_min, int* VPT, ClusterLaunch* out) {
  return dtype ? cluster_lookup_t<double>(D, DV, CPT, VPT_min, VPT, out)
               : cluster_lookup_t<float>(D, DV, CPT, VPT_min, VPT, out);
}

}  // namespace admm
