// Microbenchmark: dependent global-load latency (pointer chase) on B200,
// (a) one warp alone, (b) every SM's 32 warps chasing concurrently, and
// (c) the first load after a cooperative grid.sync().
#include <cooperative_groups.h>
#include <cstdio>
#include <vector>
#include <random>
#include <algorithm>
namespace cg = cooperative_groups;

__global__ void chase(const int* __restrict__ nxt, int steps, long long* cyc, int* sink) {
  int i = (blockIdx.x * 131 + threadIdx.x * 7919) & ((1 << 22) - 1);
  long long t0 = clock64();
  for (int s = 0; s < steps; ++s) i = __ldcg(nxt + i);
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = (t1 - t0) / steps;
  if (i == -1) sink[0] = i;
}

__global__ void after_sync(const int* __restrict__ nxt, int reps, long long* cyc, int* sink) {
  cg::grid_group g = cg::this_grid();
  int i = (blockIdx.x * 977 + threadIdx.x) & ((1 << 22) - 1);
  long long acc = 0;
  for (int r = 0; r < reps; ++r) {
    g.sync();
    long long t0 = clock64();
    i = nxt[i];
    i = nxt[i];
    long long t1 = clock64();
    acc += (t1 - t0) / 2;
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[1] = acc / reps;
  if (i == -1) sink[0] = i;
}

int main() {
  const int n = 1 << 22;  // 16 MB of ints: L2 resident
  std::vector<int> h(n);
  std::vector<int> perm(n);
  for (int k = 0; k < n; ++k) perm[k] = k;
  std::mt19937 rng(1);
  std::shuffle(perm.begin(), perm.end(), rng);
  for (int k = 0; k < n; ++k) h[perm[k]] = perm[(k + 1) % n];
  int *d, *sink; long long* cyc;
  cudaMalloc(&d, n * 4); cudaMalloc(&sink, 4); cudaMalloc(&cyc, 16);
  cudaMemcpy(d, h.data(), n * 4, cudaMemcpyHostToDevice);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long hc[2];
  chase<<<1, 1>>>(d, 4096, cyc, sink); chase<<<1, 1>>>(d, 4096, cyc, sink);
  cudaMemcpy(hc, cyc, 8, cudaMemcpyDeviceToHost);
  printf("single thread dependent load: %lld cycles\n", hc[0]);
  chase<<<sms, 1024>>>(d, 1024, cyc, sink); chase<<<sms, 1024>>>(d, 1024, cyc, sink);
  cudaMemcpy(hc, cyc, 8, cudaMemcpyDeviceToHost);
  printf("all SMs x 1024 threads chasing: %lld cycles per dependent load\n", hc[0]);
  int reps = 200; void* args[] = {&d, &reps, &cyc, &sink};
  cudaLaunchCooperativeKernel((void*)after_sync, sms, 1024, args, 0, 0);
  cudaMemcpy(hc, cyc, 16, cudaMemcpyDeviceToHost);
  printf("after grid.sync, all SMs x 1024 threads: %lld cycles per dependent load (%s)\n", hc[1],
         cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
