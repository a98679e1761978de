"""Flooding sum-product BP on the GPU: the reference-compatible API.

Mirror of ``polylp.bp_decoder`` (/root/reference/pkg/src/polylp/bp_decoder.py):

* :class:`BpConfig` -- same fields, defaults and validation (:22-34);
* :func:`posterior_llrs` ``(gamma, code, config) -> (beliefs, iterations,
  found)`` (:55-95) and :func:`decode_bp` ``(gamma, code, config) ->
  DecodeOutput`` (:98-112), computed in fp64 on the GPU;

plus the batch entry point :func:`decode_bp_batch` over the same C ABI graph
handle as the ADMM decoder (``admm_bp_decode_batch``, csrc/bp.cuh).  The BP
kernels use GPU ``tanh``/``atanh``, so fp64 results agree with the reference
to rounding (not bit for bit); the message schedule, products, clips and
stopping rule are the reference's operation by operation.

There is no CPU fallback: a missing extension raises ``RuntimeError``.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch
from numpy.typing import ArrayLike, NDArray

from . import _lib
from .admm_decoder import STATUS_CONVERGED, STATUS_MAX_ITERS, DecodeOutput, _dtype_code, _ptr, device_graph
from .codes import as_code


@dataclass(frozen=True)
class BpConfig:
    """Iteration cap, saturation magnitude (nats) and early-exit toggle (bp_decoder.py:22-34)."""

    t_max: int = 1000
    llr_clip: float = 30.0
    early_stop: bool = True

    def __post_init__(self) -> None:
        if self.t_max < 1:
            raise ValueError("t_max must be at least 1")
        if self.llr_clip <= 0:
            raise ValueError("llr_clip must be positive")


@dataclass
class BpBatchResult:
    """Per-frame results of :func:`decode_bp_batch` (device tensors)."""

    iterations: torch.Tensor             # [B] int32
    flags: torch.Tensor                  # [B] uint8: CONVERGED = early exit on a codeword
    weight: torch.Tensor                 # [B] int32
    beliefs: torch.Tensor | None = None  # [B, N] posterior LLRs
    x: torch.Tensor | None = None        # [B, N] bit-1 probabilities
    hard: torch.Tensor | None = None     # [B, N] uint8
    info: dict = field(default_factory=dict)

    @property
    def found(self) -> torch.Tensor:
        return (self.flags & _lib.ADMM_FLAG_CONVERGED) != 0

    @property
    def codeword(self) -> torch.Tensor:
        """Zero syndrome of the hard decision (used by the harness's ML accounting)."""
        return (self.flags & _lib.ADMM_FLAG_CODEWORD) != 0

    def output(self, k: int) -> DecodeOutput:
        """Frame k as the reference's :class:`DecodeOutput` (decode_bp, :98-112)."""
        if self.x is None:
            raise ValueError("decode_bp_batch was called with want_x=False")
        x = self.x[k].detach().double().cpu().numpy()
        flags = int(self.flags[k])
        hard = (self.hard[k].cpu().numpy().astype(np.uint8) if self.hard is not None
                else (self.beliefs[k].cpu().numpy() < 0.0).astype(np.uint8) if self.beliefs is not None
                else (x > 0.5).astype(np.uint8))
        return DecodeOutput(
            x=x,
            status=STATUS_CONVERGED if flags & _lib.ADMM_FLAG_CONVERGED else STATUS_MAX_ITERS,
            integral=bool(flags & _lib.ADMM_FLAG_INTEGRAL),
            iterations=int(self.iterations[k]),
            hard_decision=hard,
            ml_certificate=False,  # bp_decoder.py:111
        )


def decode_bp_batch(
    gammas,
    code,
    config: BpConfig = BpConfig(),
    *,
    dtype=torch.float64,
    device=None,
    want_beliefs: bool = True,
    want_x: bool = True,
    want_hard: bool = True,
    validate: bool = True,
    stream: torch.cuda.Stream | None = None,
) -> BpBatchResult:
    """BP-decode ``gammas`` ([B, N], one frame per row) on the GPU.

    Same conventions as :func:`paper_1204_0556_b200.decode_batch`: frames are
    independent, work is enqueued on ``stream`` without synchronising.
    """
    code = as_code(code)
    tdt = torch.float64 if _dtype_code(dtype) == _lib.ADMM_F64 else torch.float32
    dev = torch.device(device) if device is not None else (
        gammas.device if isinstance(gammas, torch.Tensor) and gammas.is_cuda else torch.device("cuda"))
    g = torch.as_tensor(gammas)
    if g.ndim == 1:
        g = g.unsqueeze(0)
    if g.ndim != 2 or g.shape[1] != code.n_vars:
        raise ValueError(f"expected a [B, {code.n_vars}] block of LLR vectors")
    g = g.to(device=dev, dtype=tdt, non_blocking=True).contiguous()
    if validate and not bool(torch.isfinite(g).all()):
        raise ValueError("LLR vector must be finite")
    B, N = g.shape[0], code.n_vars
    dg = device_graph(code, dev)
    iters = torch.empty(B, dtype=torch.int32, device=dev)
    flags = torch.empty(B, dtype=torch.uint8, device=dev)
    weight = torch.empty(B, dtype=torch.int32, device=dev)
    bel = torch.empty((B, N), dtype=tdt, device=dev) if want_beliefs else None
    x = torch.empty((B, N), dtype=tdt, device=dev) if want_x else None
    hard = torch.empty((B, N), dtype=torch.uint8, device=dev) if want_hard else None
    ws = torch.empty(16, dtype=torch.uint8, device=dev)
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    if B:
        _lib.check(_lib.load().admm_bp_decode_batch(
            dg.handle, _dtype_code(tdt), B, g.data_ptr(), N, int(config.t_max), float(config.llr_clip),
            1 if config.early_stop else 0, _ptr(bel), N, _ptr(x), N, _ptr(hard), N,
            iters.data_ptr(), flags.data_ptr(), weight.data_ptr(), ws.data_ptr(), ws.numel(), st.cuda_stream))
    res = BpBatchResult(iterations=iters, flags=flags, weight=weight, beliefs=bel, x=x, hard=hard, info=dg.info)
    res._keepalive = (g, ws)  # type: ignore[attr-defined]
    return res


def _one(gamma: ArrayLike, code, config: BpConfig) -> BpBatchResult:
    code = as_code(code)
    gamma = np.asarray(gamma, dtype=float)
    if gamma.shape != (code.n_vars,):
        raise ValueError(f"expected a length-{code.n_vars} LLR vector")
    if not np.all(np.isfinite(gamma)):
        raise ValueError("LLR vector must be finite")
    res = decode_bp_batch(gamma[None, :], code, config, dtype=torch.float64, validate=False)
    torch.cuda.current_stream().synchronize()
    return res


def posterior_llrs(gamma: ArrayLike, code, config: BpConfig = BpConfig()) -> tuple[NDArray[np.float64], int, bool]:
    """Flooding sum-product; returns (beliefs, iterations, codeword_found) (bp_decoder.py:55-95)."""
    res = _one(gamma, code, config)
    return res.beliefs[0].cpu().numpy(), int(res.iterations[0]), bool(res.found[0])


def decode_bp(gamma: ArrayLike, code, config: BpConfig = BpConfig()) -> DecodeOutput:
    """Sum-product decode; soft outputs are posterior bit-1 probabilities (bp_decoder.py:98-112)."""
    return _one(gamma, code, config).output(0)
