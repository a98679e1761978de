#include <cstdint>
#include <cstdio>
__global__ void __cluster_dims__(4,1,1) k(float* out) {
  __shared__ __align__(8) unsigned long long mbar;
  __shared__ float buf[64];
  uint32_t mb = (uint32_t)__cvta_generic_to_shared(&mbar);
  uint32_t ba = (uint32_t)__cvta_generic_to_shared(buf);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(mb), "r"(1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  uint32_t rank; asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  uint32_t dst = (rank + 1) % 4, ra, rm;
  asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(ba + 4 * threadIdx.x), "r"(dst));
  asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rm) : "r"(mb), "r"(dst));
  float v = threadIdx.x + rank;
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" :: "r"(ra), "r"(__float_as_uint(v)), "r"(rm) : "memory");
  if (threadIdx.x == 0) {
    unsigned long long st;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 %0, [%1], %2;" : "=l"(st) : "r"(mb), "r"(64 * 4) : "memory");
  }
  uint32_t done = 0;
  while (!done) {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(done) : "r"(mb), "r"(0) : "memory");
  }
  out[blockIdx.x * 64 + threadIdx.x] = buf[threadIdx.x];
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
int main() { float* d; cudaMalloc(&d, 4*64*4); k<<<4, 64>>>(d); float h[256]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost); printf("%s %f %f %f\n", cudaGetErrorString(cudaGetLastError()), h[0], h[65], h[64*3+5]); }
