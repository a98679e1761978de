// Stand-alone row-wise parity-polytope projection (project_batch,
// parity_polytope.py:352-421): one thread per row, row in registers.
#include "kernels.cuh"

namespace admm {

template <typename T, int D>
__global__ void __launch_bounds__(256) project_rows_kernel(long long m, int d, const T* __restrict__ in,
                                                            T* __restrict__ out) {
  const long long row = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (row >= m) return;
  T u[D], z[D];
#pragma unroll
  for (int k = 0; k < D; ++k) u[k] = (k < d) ? in[row * d + k] : -Num<T>::inf();
  project_pp<T, D>(u, z, d);
#pragma unroll
  for (int k = 0; k < D; ++k)
    if (k < d) out[row * d + k] = z[k];
}

template <typename T>
bool launch_project_t(int D, long long m, int d, const void* in, void* out, cudaStream_t st) {
  const int nt = 256;
  const long long grid = (m + nt - 1) / nt;
  const T* a = static_cast<const T*>(in);
  T* b = static_cast<T*>(out);
  switch (D) {
    case 4: project_rows_kernel<T, 4><<<grid, nt, 0, st>>>(m, d, a, b); return true;
    case 6: project_rows_kernel<T, 6><<<grid, nt, 0, st>>>(m, d, a, b); return true;
    case 8: project_rows_kernel<T, 8><<<grid, nt, 0, st>>>(m, d, a, b); return true;
    case 13: project_rows_kernel<T, 13><<<grid, nt, 0, st>>>(m, d, a, b); return true;
    case 16: project_rows_kernel<T, 16><<<grid, nt, 0, st>>>(m, d, a, b); return true;
    case 32: project_rows_kernel<T, 32><<<grid, nt, 0, st>>>(m, d, a, b); return true;
  }
  return false;
}

template <typename T>
__global__ void synth_kernel(long long batch, int n, SynthParams s, T* out, long long ld) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= batch * n) return;
  const long long f = idx / n;
  const int i = static_cast<int>(idx - f * n);
  out[f * ld + i] = static_cast<T>(synth_llr(s, s.trial0 + f, i));
}

void launch_synth(int dtype, long long batch, int n, const SynthParams& s, void* out, long long ld, cudaStream_t st) {
  const long long total = batch * n;
  const int nt = 256;
  const long long grid = (total + nt - 1) / nt;
  if (dtype)
    synth_kernel<double><<<grid, nt, 0, st>>>(batch, n, s, static_cast<double*>(out), ld);
  else
    synth_kernel<float><<<grid, nt, 0, st>>>(batch, n, s, static_cast<float*>(out), ld);
}

bool launch_project(int dtype, int D, long long m, int d, const void* in, void* out, cudaStream_t st) {
  return dtype ? launch_project_t<double>(D, m, d, in, out, st) : launch_project_t<float>(D, m, d, in, out, st);
}

}  // namespace admm
