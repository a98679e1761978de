// Host-side interface of the cluster engine (cluster.cu).
#pragma once

#include <cuda_runtime.h>

namespace admm {

template <typename T> struct ClusterParamsT;

// Compiled shapes: D = 6, DV = 3, 2 checks and 4 variables per thread (config 5
// and other (3,6) codes beyond one SM).  fp32 (dtype 0): C = 4 CTAs of 1024
// threads or C = 8 of 512; fp64 (dtype 1): C = 8 CTAs of 512 threads.
bool cluster_supported(int dtype, int D, int DV, int C, int CPT, int VPT);
int cluster_smem_bytes(int dtype, int NPL, int DV, int NXS, int NMS);
// Smallest slot count >= npl with a compile-time variant of the kernel (0: none).
int cluster_fixed_npl(int C, int npl);
// Active clusters per GPU for `nt` threads per CTA and `smem` bytes (0 = does not fit).
cudaError_t cluster_query(int dtype, int C, int nt, int smem, int* clusters, int* regs);
bool cluster_phase_profile(int enable, unsigned long long* out8);
cudaError_t cluster_launch(int C, const ClusterParamsT<float>& p, int clusters, int nt, int smem, cudaStream_t st);
cudaError_t cluster_launch(int C, const ClusterParamsT<double>& p, int clusters, int nt, int smem, cudaStream_t st);

}  // namespace admm
