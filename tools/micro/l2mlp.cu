// Memory-level parallelism of L2-resident gathers on B200: how long does one
// "round" of K independent coalesced 128-byte warp loads per thread take with
// a full SM (1024 threads) -- versus the same bytes moved by cp.async.bulk
// into shared memory?  (Question behind the sharded engine's slow phases.)
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(1024, 1) ld_rounds(const float* __restrict__ buf, size_t n_lines, int K, int rounds,
                                                      float* out, unsigned long long* cyc) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned long long h = (blockIdx.x * 32 + w) * 2654435761ull;
  float acc = 0.f;
  __syncthreads();
  const long long t0 = clock64();
  for (int r = 0; r < rounds; ++r) {
    float v[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      if (k < K) {
        h = h * 6364136223846793005ull + 1442695040888963407ull;
        const size_t line = (h >> 20) & (n_lines - 1);
        v[k] = __ldcg(buf + line * 32 + lane);
      }
    }
#pragma unroll
    for (int k = 0; k < 16; ++k)
      if (k < K) acc += v[k];
    __syncthreads();
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  if (acc == 12345.f) out[0] = acc;
}

__global__ void __launch_bounds__(1024, 1) bulk_rounds(const float* __restrict__ buf, size_t n_lines, int K, int rounds,
                                                        float* out, unsigned long long* cyc) {
  extern __shared__ __align__(128) float stage[];  // [K*32 lines][32]
  __shared__ __align__(8) unsigned long long bar;
  const int tid = threadIdx.x;
  const unsigned bar_a = (unsigned)__cvta_generic_to_shared(&bar);
  if (tid == 0) asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(bar_a));
  __syncthreads();
  unsigned long long h = blockIdx.x * 2654435761ull;
  const int lines = K * 32;  // same bytes as K loads by 32 warps
  float acc = 0.f;
  const long long t0 = clock64();
  for (int r = 0; r < rounds; ++r) {
    if (tid < 32) {
      if (tid == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(bar_a), "r"(lines * 128) : "memory");
      __syncwarp();
      for (int q = tid; q < lines; q += 32) {
        unsigned long long hh = (h + q) * 6364136223846793005ull + 1442695040888963407ull + r;
        const size_t line = (hh >> 20) & (n_lines - 1);
        const unsigned dst = (unsigned)__cvta_generic_to_shared(stage + q * 32);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 128, [%2];"
                     ::"r"(dst), "l"(buf + line * 32), "r"(bar_a) : "memory");
      }
    }
    // wait for phase r
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n"
        ::"r"(bar_a), "r"(r & 1) : "memory");
    for (int q = tid; q < lines * 32; q += 1024) acc += stage[q];
    __syncthreads();
  }
  const long long t1 = clock64();
  if (tid == 0) cyc[blockIdx.x] = t1 - t0;
  if (acc == 12345.f) out[0] = acc;
}

int main() {
  const size_t bytes = 16u << 20, n_lines = bytes / 128;
  float* buf;
  float* out;
  unsigned long long* cyc;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 0, bytes);
  cudaMalloc(&out, 4);
  cudaMalloc(&cyc, 148 * 8);
  unsigned long long h[148];
  const int rounds = 200;
  cudaFuncSetAttribute(bulk_rounds, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int K : {1, 2, 4, 8, 12, 16}) {
    for (int rep = 0; rep < 2; ++rep) ld_rounds<<<148, 1024>>>(buf, n_lines, K, rounds, out, cyc);
    cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double m = 0;
    for (int i = 0; i < 148; ++i) m += h[i];
    m /= 148.0 * rounds;
    const double bytes_sm = 1024.0 * K * 4;
    printf("ld.global  K=%2d: %7.0f cycles/round  %6.1f B/cycle/SM  (%d warp-lines in flight)\n", K, m, bytes_sm / m, 32 * K);
    const int smem = K * 32 * 128;
    if (smem <= 200 * 1024) {
      for (int rep = 0; rep < 2; ++rep) bulk_rounds<<<148, 1024, smem>>>(buf, n_lines, K, rounds, out, cyc);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("bulk error %s\n", cudaGetErrorString(e)); return 1; }
      cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
      m = 0;
      for (int i = 0; i < 148; ++i) m += h[i];
      m /= 148.0 * rounds;
      printf("cp.async.bulk K=%2d: %7.0f cycles/round  %6.1f B/cycle/SM\n", K, m, bytes_sm / m);
    }
  }
  return 0;
}
