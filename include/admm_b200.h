/*
 * admm_b200.h -- C ABI of the B200-native ADMM-LP decoder (sm_100a).
 *
 * This is the drop-in boundary for the reference's decoder path
 * (polylp, /root/reference/pkg/src/polylp).  The reference is pure Python and
 * has no FFI of its own; each entry point below replaces the Python function
 * named beside it, and the Python shim in paper_1204_0556_b200/ binds them
 * with ctypes (INTEGRATION.md shows the binding).
 *
 * Conventions
 *   - Every function returns 0 on success or a negative ADMM_E_* code; the
 *     thread-local message is available from admm_last_error().  No C++
 *     exception crosses this boundary.
 *   - All array arguments of admm_decode_batch / admm_project_batch are
 *     DEVICE pointers on the graph's device; the caller owns them.  Optional
 *     outputs may be NULL.  Work is enqueued on `stream` (a cudaStream_t, NULL
 *     = legacy default stream) and the call returns without synchronising.
 *   - A graph handle is immutable after creation (like ParityCheckMatrix,
 *     codes.py:28-32) and may be shared by host threads and streams.
 *   - dtype: ADMM_F32 (throughput mode) or ADMM_F64 (parity mode).
 */
#ifndef ADMM_B200_H
#define ADMM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ADMM_B200_VERSION 1

enum admm_dtype { ADMM_F32 = 0, ADMM_F64 = 1 };

enum admm_status {
  ADMM_OK = 0,
  ADMM_E_ARG = -1,         /* invalid argument (shape, range, null pointer)   */
  ADMM_E_UNSUPPORTED = -2, /* graph shape outside the compiled kernel buckets  */
  ADMM_E_CUDA = -3,        /* CUDA runtime error (message has the CUDA string) */
  ADMM_E_WORKSPACE = -4    /* workspace too small                              */
};

/* Per-frame flag bits written to flags_out. */
#define ADMM_FLAG_CONVERGED 1u /* status == "Converged" (admm_decoder.py:23)     */
#define ADMM_FLAG_INTEGRAL 2u  /* all |x - round(x)| <= 1e-5 (admm_decoder.py:96) */
#define ADMM_FLAG_CODEWORD 4u  /* hard decision satisfies every check           */

/* Engine selection for admm_graph_create_ex. */
enum admm_engine {
  ADMM_ENGINE_AUTO = 0,      /* resident if the code fits one SM, else streaming placement (cluster engine where placed) */
  ADMM_ENGINE_RESIDENT = 1,  /* one CTA per frame, state on chip (fails if it does not fit) */
  ADMM_ENGINE_STREAMING = 3, /* codes beyond one SM: sharded kernel (small batches), wide HBM kernel (>= 1024 frames) */
  ADMM_ENGINE_CLUSTER = 4,   /* streaming placement + the cluster engine required (fp32; fp64 on 8-CTA clusters) */
  ADMM_ENGINE_WIDE = 5       /* streaming placement, wide HBM-streaming kernel for every batch size */
};

/* Kernel ids reported by admm_decode_kernel. */
enum admm_kernel {
  ADMM_KERNEL_RESIDENT = 1,  /* generic resident (one CTA per frame)              */
  ADMM_KERNEL_REGULAR = 2,   /* regular-code resident                              */
  ADMM_KERNEL_SHARDED = 3,   /* sharded / L2 streaming (codes beyond one SM)       */
  ADMM_KERNEL_CLUSTER = 4,   /* cluster engine: one 8- (or 4-) CTA cluster per frame */
  ADMM_KERNEL_WIDE = 5       /* wide HBM streaming (large batches beyond one SM)   */
};

typedef struct admm_graph admm_graph;

typedef struct admm_graph_info {
  int32_t n_vars, n_checks, n_edges;
  int32_t max_check_degree, max_var_degree;
  int32_t engine;           /* 1 resident generic, 2 resident regular, 3 streaming */
  int32_t degree_bucket;    /* D: compiled check-degree bucket   */
  int32_t checks_per_thread;
  int32_t threads_per_cta;
  int32_t ctas_per_sm_f32, ctas_per_sm_f64;
  int32_t smem_bytes_f32, smem_bytes_f64;
  int32_t regs_f32, regs_f64;
  int32_t num_sms;
  int32_t cluster_size;     /* CTAs per cluster of the cluster engine (0: not placed) */
  double layout_cost_before, layout_cost_after; /* bank-conflict cost of the relabeling (engine 2) */
  int32_t cluster_active;   /* clusters resident per GPU (cluster engine) */
  int32_t cluster_threads, cluster_smem, cluster_regs;
  int64_t cluster_exchange; /* DSMEM values exchanged per iteration and frame (ghost x + messages) */
} admm_graph_info;

/* Build the device-resident Tanner graph.  Replaces the edge-array views of
 * ParityCheckMatrix (codes.py:79-115): check_ptr[n_checks+1] / edge_var[E]
 * are the reference's CSR-by-check arrays (host pointers, any variable order
 * inside a check; edges are re-sorted as codes.py:42 does). */
int admm_graph_create(int device, int32_t n_vars, int32_t n_checks, const int32_t* check_ptr,
                      const int32_t* edge_var, admm_graph** out);
/* Same, with an explicit engine (enum admm_engine). */
int admm_graph_create_ex(int device, int32_t n_vars, int32_t n_checks, const int32_t* check_ptr,
                         const int32_t* edge_var, int engine, admm_graph** out);
int admm_graph_destroy(admm_graph* g);
int admm_graph_get_info(const admm_graph* g, admm_graph_info* info);

/* Which kernel admm_decode_batch / admm_decode_synth run for `batch` frames
 * (enum admm_kernel), or a negative error code.  Codes beyond one SM switch
 * from the sharded kernel to the wide kernel at large batches. */
int admm_decode_kernel(const admm_graph* g, int dtype, int64_t batch);

/* Bytes of device workspace admm_decode_batch needs for `batch` frames. */
size_t admm_workspace_bytes(const admm_graph* g, int dtype, int64_t batch);

/* Decode `batch` independent frames.  Replaces decode(gamma, code, config)
 * (admm_decoder.py:152-182) applied frame by frame, and make_output
 * (:92-105) for the per-frame results.
 *   gamma      [batch][ld_gamma] channel costs (LLRs), dtype
 *   mu, epsilon, t_max, rho: AdmmConfig (admm_decoder.py:27-44), validated here
 *   x_out      [batch][ld_x]   final x (the iterate of the last iteration)
 *   hard_out   [batch][ld_hard] uint8 hard decision x > 0.5
 *   iters_out  [batch] int32 iterations run
 *   flags_out  [batch] uint8 ADMM_FLAG_* bits
 *   weight_out [batch] int32 Hamming weight of the hard decision
 *   z_in/lam_in [batch][ld_edge] optional initial replicas / duals in the
 *              reference edge order (NULL = zeros, AdmmState.initial)
 *   z_out/lam_out [batch][ld_edge] optional final replicas / duals
 *   workspace  device scratch of admm_workspace_bytes() bytes             */
int admm_decode_batch(const admm_graph* g, int dtype, int64_t batch, const void* gamma,
                      int64_t ld_gamma, double mu, double epsilon, int32_t t_max, double rho,
                      void* x_out, int64_t ld_x, uint8_t* hard_out, int64_t ld_hard,
                      int32_t* iters_out, uint8_t* flags_out, int32_t* weight_out,
                      const void* z_in, const void* lam_in, void* z_out, void* lam_out,
                      int64_t ld_edge, void* workspace, size_t workspace_bytes, void* stream);

/* Channel of the fused frame synthesis (channels.py:19-61); the codeword is
 * all-zero (the reference harness's default, simulator.py:252-256). */
enum admm_channel_kind { ADMM_CHANNEL_BSC = 1, ADMM_CHANNEL_AWGN = 2 };
typedef struct admm_channel {
  int32_t kind;  /* admm_channel_kind */
  double p;      /* BSC crossover probability, (0, 0.5] */
  double snr_db; /* AWGN Eb/N0 in dB */
  double rate;   /* AWGN code rate in (0, 1] (noise variance 1/(2 R 10^(snr/10))) */
} admm_channel;

/* Decode frames trial0 .. trial0+batch-1 of channel point `point` whose LLRs
 * are SYNTHESISED on the GPU from (seed, point, trial) with Philox4x32-10 --
 * the counter-based analogue of the reference harness's per-trial seeding
 * (simulator.py:169-173): a trial's LLRs never depend on the batch, engine or
 * GPU that decodes it.  Outputs as admm_decode_batch; no LLR input traffic. */
int admm_decode_synth(const admm_graph* g, int dtype, int64_t batch, const admm_channel* channel,
                      uint64_t seed, uint32_t point, int64_t trial0, double mu, double epsilon,
                      int32_t t_max, double rho, void* x_out, int64_t ld_x, uint8_t* hard_out,
                      int64_t ld_hard, int32_t* iters_out, uint8_t* flags_out, int32_t* weight_out,
                      void* workspace, size_t workspace_bytes, void* stream);

/* The same synthesised LLRs written to memory ([batch][ld] device array). */
int admm_synth_llr(int dtype, int64_t batch, int32_t n_vars, const admm_channel* channel, uint64_t seed,
                   uint32_t point, int64_t trial0, void* out, int64_t ld, void* stream);

/* Row-wise projection onto the parity polytope.  Replaces project_batch
 * (parity_polytope.py:352-421): values and out are [m][d] row-major device
 * arrays, 1 <= d <= 32. */
int admm_project_batch(int dtype, int64_t m, int32_t d, const void* values, void* out,
                       void* stream);

/* Phase profiler of the sharded engine (tracing aid): enable = 1 resets and
 * turns on clock64() accumulation in CTA 0, 0 turns it off, -1 leaves it;
 * cycles8 (host, may be NULL) receives {variable phase, grid sync, check
 * phase, grid sync, slot phase, passes, 0, 0} accumulated so far. */
int admm_phase_profile(int enable, uint64_t* cycles8);
/* Same for the wide kernel (wide.cuh): cycles8 = {variable phase, grid sync,
 * check phase, grid sync, slot phase, grid sync, passes, 0} of CTA 0. */
int admm_wide_phase_profile(int enable, uint64_t* cycles8);
/* Same for the cluster engine (cluster.cuh): cycles8 = {scatter-in, variable
 * phase, x-send, cluster barrier A, check phase, msg-send, barrier B +
 * decision, iterations} of thread 0 of CTA 0. */
int admm_cluster_phase_profile(int enable, uint64_t* cycles8);

/* Flooding sum-product BP on the same graph handle (the comparison baseline,
 * SURVEY.md 8f #4).  Replaces posterior_llrs / decode_bp
 * (bp_decoder.py:55-112) with BpConfig (t_max, llr_clip, early_stop)
 * (bp_decoder.py:22-34) for a batch of frames:
 *   gamma        [batch][ld_gamma] device LLRs (dtype)
 *   beliefs_out  [batch][ld_beliefs] posterior LLRs (may be NULL)
 *   x_out        [batch][ld_x] bit-1 probabilities 0.5 (1 - tanh(b / 2)) (may be NULL)
 *   hard_out, iters_out, flags_out, weight_out as admm_decode_batch;
 *   flags: CONVERGED = early exit on a codeword, INTEGRAL as the reference's
 *   decode_bp, CODEWORD = zero syndrome of the hard decision.
 *   workspace    >= 16 bytes of device scratch.
 * Codes whose per-frame state does not fit one SM return ADMM_E_UNSUPPORTED. */
int admm_bp_decode_batch(const admm_graph* g, int dtype, int64_t batch, const void* gamma, int64_t ld_gamma,
                         int32_t t_max, double llr_clip, int32_t early_stop, void* beliefs_out,
                         int64_t ld_beliefs, void* x_out, int64_t ld_x, uint8_t* hard_out, int64_t ld_hard,
                         int32_t* iters_out, uint8_t* flags_out, int32_t* weight_out, void* workspace,
                         size_t workspace_bytes, void* stream);

/* Step API: the reference's AdmmState driven by hand (admm_decoder.py:47-149,
 * tests/test_admm.py:147-168, 208-240), batched.  All arrays are DEVICE
 * arrays in the reference's edge order (codes.py:91-99), one frame per row:
 * edge arrays [batch][ld_edge], variable arrays [batch][ld].  In fp64 the
 * x- and lambda-updates are bit-identical to the reference's expressions
 * (true IEEE division); the z-update differs only inside the projection.
 *   admm_x_update      x_update (:108-124): x = clip((sum_e (z - lam/mu) - gamma/mu) / deg, 0, 1),
 *                      deg-0 variables take gamma < 0
 *   admm_z_update      z_update (:127-141): w = rho x[edge_var] + (1 - rho) z_old,
 *                      z_out = project(w + lam / mu) per check; w_out (may be NULL) receives w
 *   admm_lambda_update lambda_update (:144-149): lam_out = lam + mu (w - z) (lam_out may alias lam) */
int admm_x_update(const admm_graph* g, int dtype, int64_t batch, const void* z, const void* lam, int64_t ld_edge,
                  const void* gamma, int64_t ld_gamma, double mu, void* x_out, int64_t ld_x, void* stream);
int admm_z_update(const admm_graph* g, int dtype, int64_t batch, const void* x, int64_t ld_x, const void* z_old,
                  const void* lam, int64_t ld_edge, double mu, double rho, void* z_out, void* w_out, void* stream);
int admm_lambda_update(const admm_graph* g, int dtype, int64_t batch, const void* lam, const void* w, const void* z,
                       int64_t ld_edge, double mu, void* lam_out, void* stream);

/* Row-wise membership test of the parity polytope within `tol`.  Replaces
 * membership (parity_polytope.py:69-91): values [m][d] device array,
 * 1 <= d <= 32; out[m] uint8 (1 = inside). */
int admm_membership_batch(int dtype, int64_t m, int32_t d, const void* values, double tol, uint8_t* out,
                          void* stream);

const char* admm_last_error(void);
int admm_version(void);
/* Build flags: ADMM_BUILD_CHECKED = the checked build (make checked): shared-memory /
 * DSMEM bounds checks, asserts and barrier jitter compiled into the kernels. */
#define ADMM_BUILD_CHECKED 1
int admm_build_flags(void);
/* Negative control of the checked build: a one-CTA kernel that reads one word
 * past its shared memory when bad != 0 (the checked build traps; the normal
 * build reads garbage) or the last in-bounds word otherwise.  out: 1 device float. */
int admm_checked_probe(int bad, float* out, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* ADMM_B200_H */
