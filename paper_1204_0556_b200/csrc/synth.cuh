// On-GPU channel synthesis keyed by (seed, point, trial) -- SURVEY.md 8f #1.
//
// The reference harness derives every trial's frame from
// SeedSequence(seed, (point, trial)) (simulator.py:169-173) so its statistics
// do not depend on how trials are split across workers.  Here the same
// property comes from a counter-based generator: gamma_i of trial t at
// channel point k is a pure function of (seed, k, t, i) -- Philox4x32-10 with
// key (seed, k) and counter (t, i) -- so any batch, slot, engine or GPU that
// decodes trial t sees bit-identical LLRs.  Statistically this is the
// reference channel (all-zero codeword, channels.py:73-110); it is not
// numpy's PCG64 stream (parity runs use host frames for that).
//
//   BSC(p):  gamma = +log((1-p)/p), negated with probability p
//   AWGN:    y = 1 + sigma n,  gamma = 2 y / sigma^2,  n ~ N(0,1) by Box-Muller
//            (computed in fp64 for both decoder precisions, so fp32 and fp64
//            modes see the same frame up to the final cast)
#pragma once

#include <stdint.h>

namespace admm {

struct SynthParams {
  int kind;                  // 0 = none (gamma from memory), 1 = BSC, 2 = AWGN
  uint32_t seed_lo, seed_hi; // 64-bit seed
  uint32_t point;            // channel point index
  long long trial0;          // trial index of frame 0 of this call
  double bsc_p, bsc_llr;     // BSC crossover and |gamma|
  double sigma, two_over_var;
};

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
  constexpr uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(M0, c.x), lo0 = M0 * c.x;
    const uint32_t hi1 = __umulhi(M1, c.z), lo1 = M1 * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += W0;
    k.y += W1;
  }
  return c;
}

// LLR of variable i of trial `trial` (double precision).
__device__ __forceinline__ double synth_llr(const SynthParams& s, long long trial, int i) {
  const uint2 key = make_uint2(s.seed_lo ^ (s.point * 0x85EBCA6Bu), s.seed_hi + s.point);
  const uint32_t tlo = static_cast<uint32_t>(trial), thi = static_cast<uint32_t>(trial >> 32);
  if (s.kind == 1) {
    const uint4 r = philox4x32_10(make_uint4(tlo, thi, static_cast<uint32_t>(i >> 2), 0x42534331u), key);
    const uint32_t w = (i & 3) == 0 ? r.x : (i & 3) == 1 ? r.y : (i & 3) == 2 ? r.z : r.w;
    const double u = (static_cast<double>(w) + 0.5) * 2.3283064365386963e-10;  // 2^-32
    return u < s.bsc_p ? -s.bsc_llr : s.bsc_llr;
  }
  const uint4 r = philox4x32_10(make_uint4(tlo, thi, static_cast<uint32_t>(i >> 1), 0x4157474Eu), key);
  const uint64_t a = (static_cast<uint64_t>(r.x) << 21) ^ (r.y >> 11);
  const uint64_t b = (static_cast<uint64_t>(r.z) << 21) ^ (r.w >> 11);
  const double u1 = (static_cast<double>(a & ((1ull << 53) - 1)) + 0.5) * 1.1102230246251565e-16;  // 2^-53
  const double u2 = static_cast<double>(b & ((1ull << 53) - 1)) * 1.1102230246251565e-16;
  const double rad = sqrt(-2.0 * log(u1));
  double sn, cs;
  sincospi(2.0 * u2, &sn, &cs);
  const double n = (i & 1) ? rad * sn : rad * cs;
  return (1.0 + s.sigma * n) * s.two_over_var;
}

}  // namespace admm
