// Host-side interface of the BP kernels (bp.cu), kept free of device code so
// abi.cu can include it next to kernels.cuh.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "synth.cuh"

namespace admm {

struct BpGraphArgs {
  int n_vars, n_checks, m_pad;
  const int* chk_var;  // [D][m_pad] ORIGINAL variable numbering
  const uint16_t* var_pos;
  const uint8_t* var_deg;
};

struct BpFrameArgs {
  long long batch;
  const void* gamma;
  long long ld_gamma;
  double llr_clip;
  int t_max, early_stop;
  void* beliefs_out;
  long long ld_beliefs;
  void* x_out;
  long long ld_x;
  uint8_t* hard_out;
  long long ld_hard;
  int* iters_out;
  uint8_t* flags_out;
  int* weight_out;
  int* queue;
  SynthParams synth;
};

using BpLaunchFn = cudaError_t (*)(const BpGraphArgs&, const BpFrameArgs&, int grid, int nt, int smem,
                                   cudaStream_t st);

struct BpLaunch {
  const void* fn;
  BpLaunchFn launch;
  int smem, occupancy, regs;
};

bool bp_lookup(int dtype, int D, int CPT, int DVMAX, BpLaunch* out);
int bp_smem_bytes(int elem, int n_vars, int msg_len, int dvmax);

}  // namespace admm
