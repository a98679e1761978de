// Host-side launchers of the step-API and membership kernels (steps.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace admm {

// Device views of the graph in the reference's numbering (codes.py:79-115).
struct StepGraph {
  int n_vars, n_checks, m_pad, D, dv_stride;
  const int* chk_var;    // [D][m_pad] variable of slot k of check c (ascending), -1 padding
  const int* check_ptr;  // [n_checks + 1] first edge of each check
  const int* var_edge;   // [n_vars][dv_stride] edge ids of each variable, increasing
  const uint8_t* var_deg;
};

void launch_x_update(int dtype, const StepGraph& g, long long batch, const void* z, const void* lam,
                     long long ld_edge, const void* gamma, long long ld_gamma, double mu, void* x, long long ld_x,
                     cudaStream_t st);
bool launch_z_update(int dtype, const StepGraph& g, long long batch, const void* x, long long ld_x,
                     const void* z_old, const void* lam, long long ld_edge, double mu, double rho, void* z_new,
                     void* w_out, cudaStream_t st);
void launch_lambda_update(int dtype, long long batch, int n_edges, const void* lam, const void* w, const void* z,
                          long long ld_edge, double mu, void* lam_out, cudaStream_t st);
bool launch_membership(int dtype, int D, long long m, int d, const void* in, double tol, uint8_t* out,
                       cudaStream_t st);

cudaError_t launch_checked_probe(int bad, float* out, cudaStream_t st);

}  // namespace admm
