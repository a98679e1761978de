// Instantiation and launch of the cluster engine (cluster.cuh).
#include "cluster.cuh"
#include "cluster_launch.h"

#include <cstdlib>

namespace admm {

namespace {

constexpr int kD = 6, kDV = 3, kCPT = 2, kVPT = 4;
// Slot counts per part with a compiled variant (8-CTA clusters): the
// BASELINE config-5 layout has 3904 slots and is padded to the first of them.
constexpr int kNplA = 3968, kNplB = 4032;
bool g_prof = false;  // launch the profiling instantiation
const bool g_spread = std::getenv("ADMM_B200_CLUSTER_SPREAD") != nullptr;
const bool g_barrier = std::getenv("ADMM_B200_CLUSTER_BARRIER") != nullptr;  // A/B: all-to-all cluster barriers

// Instantiations: fp32 C = 4 CTAs of 1024 threads (one per SM) and C = 8 of 512
// (two per SM); fp64 C = 8 of 512 (one per SM, 128 registers).
// fns: {plain, PROF} x {cluster barriers, mbarrier syncs}
template <typename T, int C, int NT>
void fns_of(const void** fns) {
  fns[0] = reinterpret_cast<const void*>(&cluster_decode_kernel<T, kD, kDV, kCPT, kVPT, C, NT, false, false>);
  fns[1] = reinterpret_cast<const void*>(&cluster_decode_kernel<T, kD, kDV, kCPT, kVPT, C, NT, true, false>);
  fns[2] = reinterpret_cast<const void*>(&cluster_decode_kernel<T, kD, kDV, kCPT, kVPT, C, NT, false, true>);
  fns[3] = reinterpret_cast<const void*>(&cluster_decode_kernel<T, kD, kDV, kCPT, kVPT, C, NT, true, true>);
}

template <typename T>
void fixed_fns(const void** f2) {
  f2[0] = reinterpret_cast<const void*>(&cluster_decode_kernel<T, kD, kDV, kCPT, kVPT, 8, 512, false, true, kNplA>);
  f2[1] = reinterpret_cast<const void*>(&cluster_decode_kernel<T, kD, kDV, kCPT, kVPT, 8, 512, false, true, kNplB>);
}

bool fns_for(int dtype, int C, const void** fns) {
  if (dtype == 0 && C == 4) fns_of<float, 4, 1024>(fns);
  else if (dtype == 0 && C == 8) fns_of<float, 8, 512>(fns);
  else if (dtype == 1 && C == 8) fns_of<double, 8, 512>(fns);
  else return false;
  return true;
}

}  // namespace

bool cluster_supported(int dtype, int D, int DV, int C, int CPT, int VPT) {
  const void* fns[4];
  return D == kD && DV == kDV && CPT == kCPT && VPT == kVPT && fns_for(dtype, C, fns);
}

int cluster_fixed_npl(int C, int npl) {
  if (C != 8) return 0;
  return npl <= kNplA ? kNplA : npl <= kNplB ? kNplB : 0;
}

int cluster_smem_bytes(int dtype, int NPL, int DV, int NXS, int NMS) {
  return ClusterSmem(dtype ? 8 : 4, NPL, DV, NXS, NMS).total;
}

// Spread the CTAs of a cluster over distinct SMs (the hardware already does:
// tools/cluster_phases.py prints the placement).
cudaLaunchAttributeValue spread_value() {
  cudaLaunchAttributeValue v{};
  v.clusterSchedulingPolicyPreference = cudaClusterSchedulingPolicySpread;
  return v;
}

cudaError_t cluster_query(int dtype, int C, int nt, int smem, int* clusters, int* regs) {
  const void* fns[4];
  if (!fns_for(dtype, C, fns)) return cudaErrorInvalidConfiguration;
  for (const void* f : fns) {
    const cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
  }
  if (C == 8) {  // the compile-time-NPL variants share the launch shape
    const void* f2[2];
    if (dtype == 0) fixed_fns<float>(f2); else fixed_fns<double>(f2);
    for (const void* f : f2) {
      const cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (e != cudaSuccess) return e;
    }
  }
  const void* fn = fns[2];
  cudaFuncAttributes fa{};
  cudaError_t e = cudaFuncGetAttributes(&fa, fn);
  if (e != cudaSuccess) return e;
  *regs = fa.numRegs;
  if (fa.numRegs * nt > 65536) {
    *clusters = 0;
    return cudaSuccess;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(C * 64);
  cfg.blockDim = dim3(nt);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeClusterSchedulingPolicyPreference;
  attr[1].val = spread_value();
  cfg.attrs = attr;
  cfg.numAttrs = g_spread ? 2 : 1;
  return cudaOccupancyMaxActiveClusters(clusters, fn, &cfg);
}

namespace {

template <typename T, int C, int NT, bool PROF>
cudaError_t launch_t(const ClusterParamsT<T>& p, int clusters, int smem, cudaStream_t st) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(clusters * C);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  int na = 0;
  if (g_spread) {
    attr[0].id = cudaLaunchAttributeClusterSchedulingPolicyPreference;
    attr[0].val = spread_value();
    na = 1;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  // compile-time slot counts (8-CTA clusters, mbarrier syncs): the message rows
  // sit at immediate offsets from the x slots (cluster_fixed_npl)
  if constexpr (C == 8 && !PROF) {
    if (p.dense && !g_barrier) {
      if (p.NPL == kNplA) return cudaLaunchKernelEx(&cfg, cluster_decode_kernel<T, kD, kDV, kCPT, kVPT, C, NT, false, true, kNplA>, p);
      if (p.NPL == kNplB) return cudaLaunchKernelEx(&cfg, cluster_decode_kernel<T, kD, kDV, kCPT, kVPT, C, NT, false, true, kNplB>, p);
    }
  }
  if (p.dense && !g_barrier)
    return cudaLaunchKernelEx(&cfg, cluster_decode_kernel<T, kD, kDV, kCPT, kVPT, C, NT, PROF, true>, p);
  return cudaLaunchKernelEx(&cfg, cluster_decode_kernel<T, kD, kDV, kCPT, kVPT, C, NT, PROF, false>, p);
}

}  // namespace

cudaError_t cluster_launch(int C, const ClusterParamsT<float>& p, int clusters, int nt, int smem, cudaStream_t st) {
  if (nt != 4096 / C) return cudaErrorInvalidConfiguration;  // compiled CTA sizes
  cudaGetLastError();
  if (C == 8)
    return g_prof ? launch_t<float, 8, 512, true>(p, clusters, smem, st) : launch_t<float, 8, 512, false>(p, clusters, smem, st);
  return g_prof ? launch_t<float, 4, 1024, true>(p, clusters, smem, st) : launch_t<float, 4, 1024, false>(p, clusters, smem, st);
}

cudaError_t cluster_launch(int C, const ClusterParamsT<double>& p, int clusters, int nt, int smem, cudaStream_t st) {
  if (C != 8 || nt != 512) return cudaErrorInvalidConfiguration;
  cudaGetLastError();
  return g_prof ? launch_t<double, 8, 512, true>(p, clusters, smem, st) : launch_t<double, 8, 512, false>(p, clusters, smem, st);
}

bool cluster_phase_profile(int enable, unsigned long long* out8) {
  if (out8 && cudaMemcpyFromSymbol(out8, g_cl_cycles, sizeof(unsigned long long) * 8) != cudaSuccess) return false;
  if (enable >= 0) {
    const unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (cudaMemcpyToSymbol(g_cl_cycles, z, sizeof(z)) != cudaSuccess) return false;
    g_prof = enable > 0;
  }
  return true;
}

}  // namespace admm
