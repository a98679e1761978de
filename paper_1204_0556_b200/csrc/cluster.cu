// Instantiation and launch of the cluster engine (cluster.cuh).
#include "cluster.cuh"
#include "cluster_launch.h"

#include <cstdlib>

namespace admm {

namespace {

constexpr int kD = 6, kDV = 3, kCPT = 2, kVPT = 4;
bool g_prof = false;  // launch the profiling instantiation
const bool g_spread = std::getenv("ADMM_B200_CLUSTER_SPREAD") != nullptr;
const bool g_barrier = std::getenv("ADMM_B200_CLUSTER_BARRIER") != nullptr;  // A/B: all-to-all cluster barriers

// Instantiations: C = 4 CTAs of 1024 threads (one per SM), C = 8 of 512 (two per SM).
template <int C, bool PROF>
const void* fn_of() {
  return reinterpret_cast<const void*>(&cluster_decode_kernel<kD, kDV, kCPT, kVPT, C, 4096 / C, PROF>);
}

const void* kernel_fn(int C) { return C == 8 ? fn_of<8, false>() : fn_of<4, false>(); }

template <int C, int NT>
void fns_of(const void** fns) {
  fns[0] = reinterpret_cast<const void*>(&cluster_decode_kernel<kD, kDV, kCPT, kVPT, C, NT, false, false>);
  fns[1] = reinterpret_cast<const void*>(&cluster_decode_kernel<kD, kDV, kCPT, kVPT, C, NT, true, false>);
  fns[2] = reinterpret_cast<const void*>(&cluster_decode_kernel<kD, kDV, kCPT, kVPT, C, NT, false, true>);
  fns[3] = reinterpret_cast<const void*>(&cluster_decode_kernel<kD, kDV, kCPT, kVPT, C, NT, true, true>);
}

void set_smem_all(int C, int smem) {
  const void* fns[4];
  if (C == 8)
    fns_of<8, 512>(fns);
  else
    fns_of<4, 1024>(fns);
  for (const void* f : fns) cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
}

}  // namespace

bool cluster_supported(int D, int DV, int C, int CPT, int VPT) {
  return D == kD && DV == kDV && (C == 4 || C == 8) && CPT == kCPT && VPT == kVPT;
}

int cluster_smem_bytes(int NPL, int DV, int NXS, int NMS) { return ClusterSmem(NPL, DV, NXS, NMS).total; }

// Spread the CTAs of a cluster over distinct SMs (two CTAs of DIFFERENT
// clusters then share an SM at C = 8, so one hides the other's barriers).
cudaLaunchAttributeValue spread_value() {
  cudaLaunchAttributeValue v{};
  v.clusterSchedulingPolicyPreference = cudaClusterSchedulingPolicySpread;
  return v;
}

cudaError_t cluster_query(int C, int nt, int smem, int* clusters, int* regs) {
  const void* fn = kernel_fn(C);
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  set_smem_all(C, smem);
  cudaFuncAttributes fa{};
  e = cudaFuncGetAttributes(&fa, fn);
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

template <int C, int NT, bool PROF>
cudaError_t launch_t(const ClusterParams& p, int clusters, int smem, cudaStream_t st) {
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
  if (p.dense && !g_barrier)
    return cudaLaunchKernelEx(&cfg, cluster_decode_kernel<kD, kDV, kCPT, kVPT, C, NT, PROF, true>, p);
  return cudaLaunchKernelEx(&cfg, cluster_decode_kernel<kD, kDV, kCPT, kVPT, C, NT, PROF, false>, p);
}

cudaError_t cluster_launch(int C, const ClusterParams& p, int clusters, int nt, int smem, cudaStream_t st) {
  if (nt != 4096 / C) return cudaErrorInvalidConfiguration;  // compiled CTA sizes
  cudaGetLastError();
  if (C == 8) return g_prof ? launch_t<8, 512, true>(p, clusters, smem, st) : launch_t<8, 512, false>(p, clusters, smem, st);
  return g_prof ? launch_t<4, 1024, true>(p, clusters, smem, st) : launch_t<4, 1024, false>(p, clusters, smem, st);
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
