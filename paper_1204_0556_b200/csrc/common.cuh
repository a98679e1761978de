// Shared device helpers for the ADMM-LP decoder kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>
#include <cstdio>

namespace admm {

// Per-precision constants.  kTol is the facet-test tolerance: the reference's
// PARITY_TOL = 1e-9 (parity_polytope.py:19) in fp64; in fp32 the value is
// scaled to single-precision rounding (1e-9 is below one ulp of r >= 1).  The
// tolerance only decides whether a point within kTol of the facet is left
// on the cube clip, so the choice is output-continuous.
template <typename T> struct Num;
template <> struct Num<float> {
  static constexpr float kTol = 1e-6f;
  __device__ __forceinline__ static float inf() { return CUDART_INF_F; }
};
template <> struct Num<double> {
  static constexpr double kTol = 1e-9;
  __device__ __forceinline__ static double inf() { return CUDART_INF; }
};

__device__ __forceinline__ float clip01(float v) { return __saturatef(v); }  // [0,1]; -inf -> 0
// fp64 min/max as compare + select: CUDA's fmin/fmax for double carry NaN
// semantics that expand to DSETP.MIN/MAX + SEL + FSEL + LOP3 and register
// moves (~3x the instructions of the whole projection); the decoder never
// sees NaNs, and for non-NaN inputs the results are identical in value (only
// the sign of a zero may differ, which no later operation observes).
__device__ __forceinline__ double clip01(double v) { return v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v); }
__device__ __forceinline__ float vmax(float a, float b) { return fmaxf(a, b); }
__device__ __forceinline__ float vmin(float a, float b) { return fminf(a, b); }
__device__ __forceinline__ double vmax(double a, double b) { return a > b ? a : b; }
__device__ __forceinline__ double vmin(double a, double b) { return a < b ? a : b; }

// Compare-exchange primitives used by the generated sorting networks.
template <typename T> __device__ __forceinline__ void ce_desc(T& a, T& b) {
  const T hi = vmax(a, b), lo = vmin(a, b);
  a = hi;
  b = lo;
}
template <typename T> __device__ __forceinline__ void ce_asc(T& a, T& b) {
  const T lo = vmin(a, b), hi = vmax(a, b);
  a = lo;
  b = hi;
}
// fp64: one comparison drives both selects
template <> __device__ __forceinline__ void ce_desc<double>(double& a, double& b) {
  const bool sw = a < b;
  const double hi = sw ? b : a, lo = sw ? a : b;
  a = hi;
  b = lo;
}
template <> __device__ __forceinline__ void ce_asc<double>(double& a, double& b) {
  const bool sw = b < a;
  const double lo = sw ? b : a, hi = sw ? a : b;
  a = lo;
  b = hi;
}

// Rounded arithmetic.  fp64 is the parity mode: products and sums are kept
// separate (no FMA contraction) so every update reproduces the reference's
// numpy expression tree operation by operation.  fp32 is the throughput mode
// and lets the compiler contract to FFMA.
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return a * b; }
__device__ __forceinline__ float add_rn(float a, float b) { return a + b; }
__device__ __forceinline__ float sub_rn(float a, float b) { return a - b; }
__device__ __forceinline__ float div_rn(float a, float b) { return __fdividef(a, b); }

// Packed fp32 pair arithmetic (sm_100 FADD2/FMUL2/FFMA2): the same IEEE
// round-to-nearest operation in each lane, one instruction for two edges.
__device__ __forceinline__ float2 fsub2_rn(float2 a, float2 b) {
  unsigned long long ra, rb, rd;
  asm("mov.b64 %0, {%1, %2};" : "=l"(ra) : "f"(a.x), "f"(a.y));
  asm("mov.b64 %0, {%1, %2};" : "=l"(rb) : "f"(b.x), "f"(b.y));
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(rd) : "l"(ra), "l"(rb));
  float2 d;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(d.x), "=f"(d.y) : "l"(rd));
  return d;
}

// Butterfly all-reduce inside a warp.  IEEE addition is commutative, so every
// lane ends with a bitwise identical sum (lane i adds a_i + a_j, lane j adds
// a_j + a_i at each level): the convergence decision is uniform.
template <typename T> __device__ __forceinline__ T warp_allsum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---------------------------------------------------------------------------
// Checked build (make checked -> libadmm_b200_checked.so, -DADMM_CHECKED):
// compute-sanitizer is closed on the GPU pool, so the kernels carry their own
// instrumentation, compiled in only here:
//   * every bare shared-memory access (lds*/sts*) and every DSMEM address
//     (cl_addr) is bounds-checked against the CTA's shared window
//     (static + dynamic, %dynamic_smem_size), and the cluster rank against
//     the cluster size; a violation prints the address and traps;
//   * ADMM_JITTER() sleeps a pseudo-random 0-1 us per warp at the phase
//     boundaries of the barrier-synchronous kernels, so a missing barrier
//     turns into wrong or nondeterministic results in the parity tests.
// ---------------------------------------------------------------------------
#ifdef ADMM_CHECKED
extern __shared__ __align__(16) unsigned char admm_dyn_smem[];
__device__ __forceinline__ uint32_t admm_smem_end() {
  uint32_t dyn;
  asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
  return static_cast<uint32_t>(__cvta_generic_to_shared(admm_dyn_smem)) + dyn;
}
__device__ __forceinline__ void admm_check_smem(uint32_t a, uint32_t bytes) {
  if (a + bytes > admm_smem_end() || (a & (bytes - 1)) != 0) {
    printf("ADMM_CHECKED: shared access [%u, +%u) outside [0, %u) or misaligned (block %d thread %d)\n", a, bytes,
           admm_smem_end(), blockIdx.x, threadIdx.x);
    __trap();
  }
}
#define ADMM_CHECK_SMEM(a, bytes) admm::admm_check_smem((a), (bytes))
#define ADMM_ASSERT(cond)                                                                          \
  do {                                                                                             \
    if (!(cond)) {                                                                                 \
      printf("ADMM_CHECKED: %s:%d assertion %s failed (block %d thread %d)\n", __FILE__, __LINE__, #cond, \
             blockIdx.x, threadIdx.x);                                                             \
      __trap();                                                                                    \
    }                                                                                              \
  } while (0)
__device__ __forceinline__ void admm_jitter() {
  uint32_t x = static_cast<uint32_t>(clock64()) ^ (blockIdx.x * 0x9E3779B9u) ^ ((threadIdx.x >> 5) * 0x85EBCA6Bu);
  x ^= x >> 15;
  x *= 0x2C1B3C6Du;
  x ^= x >> 12;
  __nanosleep(x & 1023u);
}
#define ADMM_JITTER() admm::admm_jitter()
#else
#define ADMM_CHECK_SMEM(a, bytes) ((void)0)
#define ADMM_ASSERT(cond) ((void)0)
#define ADMM_JITTER() ((void)0)
#endif

// 32-bit shared-memory addressing.  Addresses are computed once (per CTA or
// per frame) and kept in registers, so the hot loops issue bare LDS/STS with
// no generic-to-shared conversion.  The "memory" clobber keeps the compiler
// from moving them across __syncthreads().
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ float lds(uint32_t a, float) {
  ADMM_CHECK_SMEM(a, 4);
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ double lds(uint32_t a, double) {
  ADMM_CHECK_SMEM(a, 8);
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts(uint32_t a, float v) {
  ADMM_CHECK_SMEM(a, 4);
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}
__device__ __forceinline__ void sts(uint32_t a, double v) {
  ADMM_CHECK_SMEM(a, 8);
  asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
// Four adjacent fp32 words (16-byte aligned address).
__device__ __forceinline__ float4 lds4(uint32_t a) {
  ADMM_CHECK_SMEM(a, 16);
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts4(uint32_t a, float4 v) {
  ADMM_CHECK_SMEM(a, 16);
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}
// Two adjacent fp64 words (16-byte aligned address).
__device__ __forceinline__ double2 lds2d(uint32_t a) {
  ADMM_CHECK_SMEM(a, 16);
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts2d(uint32_t a, double2 v) {
  ADMM_CHECK_SMEM(a, 16);
  asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(v.x), "d"(v.y) : "memory");
}
// Two adjacent fp32 words (8-byte aligned address).
__device__ __forceinline__ float2 lds2(uint32_t a) {
  ADMM_CHECK_SMEM(a, 8);
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts2(uint32_t a, float2 v) {
  ADMM_CHECK_SMEM(a, 8);
  asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(a), "f"(v.x), "f"(v.y) : "memory");
}

}  // namespace admm
