// DSMEM micro-benchmark for the cluster engine design (4-CTA clusters,
// 1024 threads per CTA, one CTA per SM): per-SM throughput of scattered
// 4-byte ld/st.shared::cluster (local window and remote CTAs) against plain
// LDS/STS, and the cost of a cluster barrier.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dsmem dsmem.cu && ./dsmem
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t r) {
  uint32_t o;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
  return o;
}
__device__ __forceinline__ float ldc(uint32_t a) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void stc(uint32_t a, float v) {
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}
__device__ __forceinline__ float lds(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts(uint32_t a, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}
__device__ __forceinline__ void cbar() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t crank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t hash(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

constexpr int K = 12;       // accesses per thread per iteration (2 checks x 6 edges)
constexpr int WORDS = 16384;  // 64 KB of fp32 per CTA

// MODE 0: LDS/STS local; 1: shared::cluster, own CTA only; 2: shared::cluster,
// remote with probability premote/100; 3: local LDS gathers, stores to a
// remote CTA at CONSECUTIVE addresses across the warp (coalesced, 4 B per
// lane); 4: same with 16 B per lane (v4); BAR: a cluster barrier per
// iteration (and a __syncthreads otherwise)
template <int MODE, bool BAR>
__global__ void __cluster_dims__(4, 1, 1) __launch_bounds__(1024, 1) bench(int iters, int premote, unsigned long long* out, float* sink) {
  extern __shared__ float sm[];
  const uint32_t r = crank(), base = (uint32_t)__cvta_generic_to_shared(sm);
  for (int i = threadIdx.x; i < WORDS; i += blockDim.x) sm[i] = 1.0f;
  uint32_t ga[K], sa[K];
  const uint32_t tid = blockIdx.x * 1024 + threadIdx.x;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const uint32_t h = hash(tid * 131 + k), h2 = hash(h);
    const uint32_t word = h % (WORDS / 2), word2 = WORDS / 2 + h2 % (WORDS / 2);
    uint32_t dst = r;
    if (MODE == 2 && (h2 >> 8) % 100 < (uint32_t)premote) dst = (r + 1 + (h2 >> 20) % 3) % 4;
    if (MODE == 0) {
      ga[k] = base + 4 * word;
      sa[k] = base + 4 * word2;
    } else if (MODE >= 3) {
      ga[k] = base + 4 * word;
      const uint32_t w = threadIdx.x >> 5, l = threadIdx.x & 31;
      const uint32_t off = MODE == 3 ? (WORDS / 2 + ((w * K + k) * 32 + l) % (WORDS / 2))
                                     : (WORDS / 2 + ((w * K + k) * 128 + 4 * l) % (WORDS / 2));
      sa[k] = mapa(base + 4 * off, (r + 1 + k % 3) % 4);
    } else {
      ga[k] = mapa(base + 4 * word, dst);
      sa[k] = mapa(base + 4 * word2, dst);
    }
  }
  cbar();
  float acc = 0.f;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    float v[K];
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = (MODE == 0 || MODE >= 3) ? lds(ga[k]) : ldc(ga[k]);
#pragma unroll
    for (int k = 0; k < K; ++k) acc += v[k];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (MODE == 0) sts(sa[k], acc * (k + 1));
      else if (MODE == 4) {
        const float a = acc * (k + 1);
        asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(sa[k]), "f"(a), "f"(a), "f"(a), "f"(a) : "memory");
      } else stc(sa[k], acc * (k + 1));
    }
    if (BAR) cbar();
    else __syncthreads();
  }
  long long t1 = clock64();
  cbar();
  if (threadIdx.x == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
  if (acc == 12345.f) sink[tid] = acc;
}

template <int MODE, bool BAR>
void run(const char* name, int premote, int nblocks) {
  const int iters = 2000;
  unsigned long long* d;
  float* sink;
  cudaMalloc(&d, nblocks * sizeof(unsigned long long));
  cudaMalloc(&sink, nblocks * 1024 * sizeof(float));
  cudaFuncSetAttribute(bench<MODE, BAR>, cudaFuncAttributeMaxDynamicSharedMemorySize, WORDS * 4);
  bench<MODE, BAR><<<nblocks, 1024, WORDS * 4>>>(10, premote, d, sink);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  bench<MODE, BAR><<<nblocks, 1024, WORDS * 4>>>(iters, premote, d, sink);
  cudaEventRecord(b);
  cudaError_t e = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  unsigned long long* h = new unsigned long long[nblocks];
  cudaMemcpy(h, d, nblocks * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int i = 0; i < nblocks; ++i) mean += h[i];
  mean /= nblocks;
  // per SM per iteration: 32 warps x (K loads + K stores)
  printf("%-34s premote=%3d%%  %s  %8.1f cycles/iter  %6.2f cycles per warp-access  (%.3f ms)\n", name, premote,
         e == cudaSuccess ? "ok " : cudaGetErrorString(e), mean / iters, mean / iters / (32.0 * 2 * K), ms);
  delete[] h;
  cudaFree(d);
  cudaFree(sink);
}

int main() {
  int clusters = 0;
  {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(4 * 64);
    cfg.blockDim = dim3(1024);
    cfg.dynamicSmemBytes = WORDS * 4;
    cudaFuncSetAttribute(bench<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, WORDS * 4);
    cudaOccupancyMaxActiveClusters(&clusters, (void*)bench<2, true>, &cfg);
  }
  printf("max active 4-CTA clusters (1024 threads, 64 KB smem): %d\n", clusters);
  const int nb = 4 * (clusters > 0 ? clusters : 32);
  run<0, false>("LDS/STS + syncthreads", 0, nb);
  run<1, false>("cluster window, own CTA", 0, nb);
  run<2, false>("cluster, remote", 28, nb);
  run<2, false>("cluster, remote", 75, nb);
  run<3, false>("LDS + coalesced remote STS (4 B)", 100, nb);
  run<4, false>("LDS + coalesced remote STS.v4 (16 B)", 100, nb);
  run<0, true>("LDS/STS + cluster barrier", 0, nb);
  run<2, true>("cluster, remote + cluster barrier", 28, nb);
  return 0;
}
