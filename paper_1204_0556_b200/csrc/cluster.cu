// Instantiation and launch of the cluster engine (cluster.cuh).
#include "cluster.cuh"
#include "cluster_launch.h"

namespace admm {

namespace {

constexpr int kD = 6, kDV = 3, kCPT = 2, kVPT = 4;
bool g_prof = false;  // launch the profiling instantiation

const void* kernel_fn(int C) {
  if (C == 8) return reinterpret_cast<const void*>(&cluster_decode_kernel<kD, kDV, kCPT, kVPT, 8>);
  return reinterpret_cast<const void*>(&cluster_decode_kernel<kD, kDV, kCPT, kVPT, 4>);
}

}  // namespace

bool cluster_supported(int D, int DV, int C, int CPT, int VPT) {
  return D == kD && DV == kDV && (C == 4 || C == 8) && CPT == kCPT && VPT == kVPT;
}

int cluster_smem_bytes(int NPL, int DV, int NIN, int NXS, int NMS) { return ClusterSmem(NPL, DV, NIN, NXS, NMS).total; }

cudaError_t cluster_query(int C, int nt, int smem, int* clusters, int* regs) {
  const void* fn = kernel_fn(C);
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  for (const void* pf : {reinterpret_cast<const void*>(&cluster_decode_kernel<kD, kDV, kCPT, kVPT, 4, true>),
                         reinterpret_cast<const void*>(&cluster_decode_kernel<kD, kDV, kCPT, kVPT, 8, true>)})
    cudaFuncSetAttribute(pf, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
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
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaOccupancyMaxActiveClusters(clusters, fn, &cfg);
}

cudaError_t cluster_launch(int C, const ClusterParams& p, int clusters, int nt, int smem, cudaStream_t st) {
  if (C == 8 && g_prof)
    cluster_decode_kernel<kD, kDV, kCPT, kVPT, 8, true><<<clusters * 8, nt, smem, st>>>(p);
  else if (C == 8)
    cluster_decode_kernel<kD, kDV, kCPT, kVPT, 8><<<clusters * 8, nt, smem, st>>>(p);
  else if (g_prof)
    cluster_decode_kernel<kD, kDV, kCPT, kVPT, 4, true><<<clusters * 4, nt, smem, st>>>(p);
  else
    cluster_decode_kernel<kD, kDV, kCPT, kVPT, 4><<<clusters * 4, nt, smem, st>>>(p);
  return cudaGetLastError();
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
