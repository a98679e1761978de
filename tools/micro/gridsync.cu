// Microbenchmark: cost of cooperative_groups grid.sync() on this GPU with one
// 512-thread CTA per SM (the sharded engine's launch shape).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k(int iters, int* out) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < iters; ++i) g.sync();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = iters;
}
__global__ void k_bar(int iters, unsigned* bar, int nblk) {
  // hand-rolled barrier: one atomic per CTA + spin on a generation word
  volatile unsigned* gen = bar + 1;
  for (int i = 0; i < iters; ++i) {
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned g0 = *gen;
      __threadfence();
      if (atomicAdd(bar, 1) == (unsigned)(nblk - 1)) {
        bar[0] = 0;
        __threadfence();
        atomicAdd((unsigned*)gen, 1);
      } else {
        while (*gen == g0) { __nanosleep(32); }
      }
      __threadfence();
    }
    __syncthreads();
  }
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int* out; cudaMalloc(&out, 4);
  unsigned* bar; cudaMalloc(&bar, 8); cudaMemset(bar, 0, 8);
  for (int nt : {256, 512}) {
    int iters = 10000;
    void* args[] = {&iters, &out};
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaLaunchCooperativeKernel((void*)k, sms, nt, args, 0, 0);
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)k, sms, nt, args, 0, 0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("grid.sync  %d CTAs x %d threads: %.3f us per sync\n", sms, nt, ms * 1000 / iters);
    int nb = sms;
    void* args2[] = {&iters, &bar, &nb};
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)k_bar, sms, nt, args2, 0, 0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("hand barrier %d CTAs x %d threads: %.3f us per sync (%s)\n", sms, nt, ms * 1000 / iters, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
