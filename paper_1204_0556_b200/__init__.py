"""B200-native ADMM-LP decoder for binary LDPC codes (arXiv 1204.0556).

Drop-in for the decoder path of the reference package ``polylp``
(/root/reference/pkg/src/polylp/__init__.py:8-97): the decoder names
``AdmmConfig``, ``AdmmState``, ``DecodeOutput``, ``STATUS_*``, ``decode``,
``x_update``/``z_update``/``lambda_update``, ``ParityCheckMatrix``,
``is_codeword``, ``project_batch`` and ``membership`` are exported
with the reference's signatures; the arithmetic runs in hand-written sm_100a
CUDA kernels behind the C ABI of ``include/admm_b200.h``.
"""

from .admm_decoder import (
    INTEGRALITY_TOL,
    STATUS_CONVERGED,
    STATUS_MAX_ITERS,
    AdmmConfig,
    AdmmState,
    BatchResult,
    DecodeOutput,
    decode,
    decode_batch,
    decode_synth,
    device_graph,
    lambda_update,
    make_output,
    synth_llr,
    run_iterations,
    x_update,
    z_update,
)
from .bp_decoder import BpBatchResult, BpConfig, decode_bp, decode_bp_batch, posterior_llrs
from .channels import Awgn, Bsc, llr, transmit, trial_gamma, trial_gammas
from .codes import (
    AlistParseError,
    CodeGenerationError,
    ParityCheckMatrix,
    baseline_code,
    emit_alist,
    gen_regular_ldpc,
    is_codeword,
    make_ldpc,
    parse_alist,
)
from .parity_polytope import PARITY_TOL, membership, membership_batch, project_batch
from .simulator import DecoderRef, MlOutcome, TrialStats, ml_account, run_point, stats_to_csv, sweep

__version__ = "0.1.0"

__all__ = [
    "AdmmConfig", "AdmmState", "BatchResult", "DecodeOutput", "INTEGRALITY_TOL", "STATUS_CONVERGED",
    "STATUS_MAX_ITERS", "decode", "decode_batch", "decode_synth", "device_graph", "synth_llr", "run_iterations",
    "make_output", "x_update", "z_update", "lambda_update",
    "BpBatchResult", "BpConfig", "decode_bp", "decode_bp_batch", "posterior_llrs",
    "Awgn", "Bsc", "llr", "transmit", "trial_gamma", "trial_gammas",
    "AlistParseError", "CodeGenerationError", "ParityCheckMatrix", "baseline_code", "emit_alist",
    "gen_regular_ldpc", "is_codeword", "make_ldpc", "parse_alist",
    "PARITY_TOL", "membership", "membership_batch", "project_batch",
    "DecoderRef", "MlOutcome", "TrialStats", "ml_account", "run_point", "stats_to_csv", "sweep",
]
