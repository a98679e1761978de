// DSMEM bulk-copy probe: cp.async.bulk shared::cta -> shared::cluster with
// mbarrier completion, against per-thread st.async, on 4-CTA clusters (one CTA
// of 1024 threads per SM, 33 clusters).  Each CTA sends TOTAL bytes per
// iteration, split evenly over the 3 other CTAs in runs of RUN bytes, and
// waits for the bytes it receives.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dsmem_bulk dsmem_bulk.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t r) {
  uint32_t o;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
  return o;
}
__device__ __forceinline__ void cbar() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t mb, uint32_t par) {
  uint32_t done = 0;
  for (uint32_t k = 0; !done; ++k) {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done) : "r"(mb), "r"(par) : "memory");
    if (k > (1u << 22)) __trap();  // never hang the GPU
  }
}

constexpr int SRC = 0, DST = 16384, SMEM = 32768 + 64;

// MODE 0: st.async 4 B per lane, coalesced; MODE 1: cp.async.bulk runs of RUN bytes
template <int MODE, int RUN, int TOTAL = 12288>  // TOTAL: bytes sent per CTA per iteration (a third to each peer)
__global__ void __cluster_dims__(4, 1, 1) __launch_bounds__(1024, 1) bench(int iters, unsigned long long* out, float* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint32_t rank;
  asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm), mb0 = base + 32768;
  for (int i = threadIdx.x; i < 8192; i += 1024) reinterpret_cast<float*>(sm)[i] = 1.f + i;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mb0), "r"(1) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mb0 + 8), "r"(1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  cbar();
  const int per_peer = TOTAL / 3;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    // two mbarriers by iteration parity: a CTA can run at most one iteration ahead of a peer
    const uint32_t mb = mb0 + 8 * (it & 1);
    if (MODE == 0) {
      for (int i = threadIdx.x; i < TOTAL / 4; i += 1024) {
        const uint32_t peer = (rank + 1 + i / (per_peer / 4)) & 3;
        const uint32_t off = 4 * (i % (per_peer / 4)) + rank * per_peer;
        const float v = reinterpret_cast<float*>(sm)[i];
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(mapa(base + DST + off, peer)),
                     "r"(__float_as_uint(v)), "r"(mapa(mb, peer)) : "memory");
      }
    } else {
      // generic-proxy writes of the source must be visible to the async proxy
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      const int nrun = TOTAL / RUN, rpp = per_peer / RUN;
      for (int r = threadIdx.x; r < nrun; r += 1024) {
        const uint32_t peer = (rank + 1 + r / rpp) & 3;
        const uint32_t off = RUN * (r % rpp) + rank * per_peer;
        asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         mapa(base + DST + off, peer)),
                     "r"(base + SRC + RUN * r), "r"(RUN), "r"(mapa(mb, peer)) : "memory");
      }
    }
    if (threadIdx.x == 0) {
      unsigned long long st;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 %0, [%1], %2;" : "=l"(st) : "r"(mb), "r"(TOTAL) : "memory");
    }
    mbar_wait(mb, (it >> 1) & 1);
    // consume something so iterations are ordered like the engine's
    if (threadIdx.x < 32) reinterpret_cast<float*>(sm)[threadIdx.x] += reinterpret_cast<float*>(sm + DST)[threadIdx.x];
    __syncthreads();
  }
  long long t1 = clock64();
  cbar();
  if (threadIdx.x == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
  if (reinterpret_cast<float*>(sm)[threadIdx.x] == 12345.f) sink[threadIdx.x] = 1.f;
}

template <int MODE, int RUN, int TOTAL = 12288>
void run(const char* name) {
  const int iters = 2000, nblocks = 33 * 4;
  unsigned long long* d;
  float* sink;
  cudaMalloc(&d, nblocks * sizeof(unsigned long long));
  cudaMalloc(&sink, 4096);
  cudaFuncSetAttribute(bench<MODE, RUN, TOTAL>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
  bench<MODE, RUN, TOTAL><<<nblocks, 1024, SMEM>>>(10, d, sink);
  bench<MODE, RUN, TOTAL><<<nblocks, 1024, SMEM>>>(iters, d, sink);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[33 * 4];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int i = 0; i < nblocks; ++i) mean += h[i];
  mean /= nblocks;
  printf("%-40s %6d B  %s %8.1f cycles/iter  %6.2f B/cycle sent per SM\n", name, TOTAL, e == cudaSuccess ? "ok " : cudaGetErrorString(e),
         mean / iters, TOTAL / (mean / iters));
  fflush(stdout);
  cudaFree(d);
  cudaFree(sink);
}

int main() {
  run<0, 4, 384>("st.async 4 B/lane coalesced");
  run<0, 4, 1536>("st.async 4 B/lane coalesced");
  run<0, 4, 6144>("st.async 4 B/lane coalesced");
  run<0, 4>("st.async 4 B/lane coalesced");
  run<1, 64>("cp.async.bulk runs of 64 B");
  run<1, 128>("cp.async.bulk runs of 128 B");
  run<1, 256>("cp.async.bulk runs of 256 B");
  run<1, 512>("cp.async.bulk runs of 512 B");
  run<1, 1024>("cp.async.bulk runs of 1024 B");
  run<1, 4096>("cp.async.bulk runs of 4096 B");
  return 0;
}
