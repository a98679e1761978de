// Host-side interface of the cluster engine (cluster.cu).
#pragma once

#include <cuda_runtime.h>

namespace admm {

struct ClusterParams;

// Compiled shapes: D = 6, DV = 3, C = 4 or 8 CTAs per cluster, 2 checks and
// 4 variables per thread (config 5 and other (3,6) codes beyond one SM).
bool cluster_supported(int D, int DV, int C, int CPT, int VPT);
int cluster_smem_bytes(int NPL, int DV, int NXS, int NMS);
// Active clusters per GPU for `nt` threads per CTA and `smem` bytes (0 = does not fit).
cudaError_t cluster_query(int C, int nt, int smem, int* clusters, int* regs);
bool cluster_phase_profile(int enable, unsigned long long* out8);
cudaError_t cluster_launch(int C, const ClusterParams& p, int clusters, int nt, int smem, cudaStream_t st);

}  // namespace admm
