// Instantiation and launch of the cluster engine (cluster.cuh).
#include "cluster.cuh"
#include "cluster_launch.h"

namespace admm {

namespace {

constexpr int kD = 6, kDV = 3, kCPT = 2, kVPT = 4, kC = 4;

const void* kernel_fn() { return reinterpret_cast<const void*>(&cluster_decode_kernel<kD, kDV, kCPT, kVPT, kC>); }

}  // namespace

bool cluster_supported(int D, int DV, int C, int CPT, int VPT) {
  return D == kD && DV == kDV && C == kC && CPT == kCPT && VPT == kVPT;
}

int cluster_smem_bytes(int NPL, int DV, int NIN, int NXS, int NMS) { return ClusterSmem(NPL, DV, NIN, NXS, NMS).total; }

cudaError_t cluster_query(int nt, int smem, int* clusters, int* regs) {
  const void* fn = kernel_fn();
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  cudaFuncAttributes fa{};
  e = cudaFuncGetAttributes(&fa, fn);
  if (e != cudaSuccess) return e;
  *regs = fa.numRegs;
  if (fa.numRegs * nt > 65536) {
    *clusters = 0;
    return cudaSuccess;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(kC * 64);
  cfg.blockDim = dim3(nt);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kC;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaOccupancyMaxActiveClusters(clusters, fn, &cfg);
}

cudaError_t cluster_launch(const ClusterParams& p, int clusters, int nt, int smem, cudaStream_t st) {
  cluster_decode_kernel<kD, kDV, kCPT, kVPT, kC><<<clusters * kC, nt, smem, st>>>(p);
  return cudaGetLastError();
}

}  // namespace admm
