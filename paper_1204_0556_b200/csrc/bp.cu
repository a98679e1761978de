// Instantiation table and launchers of the BP kernel (bp.cuh).
#include "bp_launch.h"

#include "bp.cuh"

namespace admm {

template <typename T, int D, int CPT, int DVMAX>
cudaError_t bp_launch_t(const BpGraphArgs& g, const BpFrameArgs& a, int grid, int nt, int smem, cudaStream_t st) {
  BpParams<T> p;
  p.n_vars = g.n_vars;
  p.n_checks = g.n_checks;
  p.m_pad = g.m_pad;
  p.chk_var = g.chk_var;
  p.var_pos = g.var_pos;
  p.var_deg = g.var_deg;
  p.batch = a.batch;
  p.gamma = static_cast<const T*>(a.gamma);
  p.ld_gamma = a.ld_gamma;
  p.clip = static_cast<T>(a.llr_clip);
  p.half_clip = static_cast<T>(0.5 * a.llr_clip);  // bp_decoder.py:41, 0.5 * clip in double
  p.guard = static_cast<T>(1.0 - 1e-15);           // _ATANH_GUARD (bp_decoder.py:19)
  p.t_max = a.t_max;
  p.early_stop = a.early_stop;
  p.beliefs_out = static_cast<T*>(a.beliefs_out);
  p.ld_beliefs = a.ld_beliefs;
  p.x_out = static_cast<T*>(a.x_out);
  p.ld_x = a.ld_x;
  p.hard_out = a.hard_out;
  p.ld_hard = a.ld_hard;
  p.iters_out = a.iters_out;
  p.flags_out = a.flags_out;
  p.weight_out = a.weight_out;
  p.queue = a.queue;
  p.synth = a.synth;
  bp_decode_kernel<T, D, CPT, DVMAX><<<grid, nt, smem, st>>>(p);
  return cudaGetLastError();
}

template <typename T, int D, int CPT, int DVMAX>
BpLaunch bp_entry() {
  return BpLaunch{reinterpret_cast<const void*>(&bp_decode_kernel<T, D, CPT, DVMAX>), &bp_launch_t<T, D, CPT, DVMAX>,
                  0, 0, 0};
}

template <typename T, int D>
bool bp_lookup_d(int CPT, int DVMAX, BpLaunch* out) {
  if (DVMAX == 4) {
    if (CPT == 1) { *out = bp_entry<T, D, 1, 4>(); return true; }
    if (CPT == 2) { *out = bp_entry<T, D, 2, 4>(); return true; }
  } else if (DVMAX == 8) {
    if (CPT == 1) { *out = bp_entry<T, D, 1, 8>(); return true; }
    if (CPT == 2) { *out = bp_entry<T, D, 2, 8>(); return true; }
  }
  return false;
}

template <typename T>
bool bp_lookup_t(int D, int CPT, int DVMAX, BpLaunch* out) {
  switch (D) {
    case 4: return bp_lookup_d<T, 4>(CPT, DVMAX, out);
    case 6: return bp_lookup_d<T, 6>(CPT, DVMAX, out);
    case 8: return bp_lookup_d<T, 8>(CPT, DVMAX, out);
    case 13: return bp_lookup_d<T, 13>(CPT, DVMAX, out);
    case 16: return bp_lookup_d<T, 16>(CPT, DVMAX, out);
    case 32: return CPT == 1 && bp_lookup_d<T, 32>(1, DVMAX, out);
  }
  return false;
}

bool bp_lookup(int dtype, int D, int CPT, int DVMAX, BpLaunch* out) {
  return dtype ? bp_lookup_t<double>(D, CPT, DVMAX, out) : bp_lookup_t<float>(D, CPT, DVMAX, out);
}

int bp_smem_bytes(int elem, int n_vars, int msg_len, int dvmax) { return BpSmem(elem, n_vars, msg_len, dvmax).total; }

}  // namespace admm
