"""Batched Monte-Carlo harness on the GPU decoder.

Mirror of ``polylp.simulator`` (/root/reference/pkg/src/polylp/simulator.py):
``DecoderRef`` (:53-72), ``MlOutcome``/``ml_account`` (:75-106),
``TrialStats`` with ``merge`` (:109-153), ``run_point`` (:223-318) with the
fixed-count and target-errors modes (exact truncation at the trial that met
the target, :286-294), ``sweep`` (:321-352) and ``stats_to_csv`` with the
same 18 columns and number formatting (:29-48, :355-394).

What changes is the execution: trials are decoded in GPU batches instead of
one ``decode`` call per trial in a process pool.  Two frame sources:

* ``frames="reference"`` (default): each trial's LLRs come from
  ``SeedSequence(entropy=seed, spawn_key=(point, trial))`` exactly as the
  reference harness draws them (simulator.py:169-173), so with the fp64
  decoder the statistics -- and the CSV with ``timing=False`` -- are the
  reference's;
* ``frames="device"``: LLRs are synthesised inside the decode kernel from
  (seed, point, trial) (csrc/synth.cuh) -- no host work and no LLR traffic,
  statistically the same channel, not bit-identical to numpy.

In both modes a trial's result depends only on (seed, point, trial), never on
the batch size or the number of GPUs.  ``DecoderRef("admm")`` and
``DecoderRef("bp")`` (flooding sum-product, csrc/bp.cuh) run on the GPU;
``("dual-ascent")`` raises (that reference baseline is out of scope).  Timing columns report each trial's share of its
batch's wall time.
"""

from __future__ import annotations

import csv
import enum
import io
import time
from dataclasses import dataclass, replace
from typing import Callable, Sequence

import numpy as np
import torch
from numpy.typing import ArrayLike, NDArray

from .admm_decoder import AdmmConfig, DecodeOutput, decode, decode_batch, decode_synth, synth_llr
from .bp_decoder import BpConfig, decode_bp, decode_bp_batch
from .channels import Awgn, Bsc, ChannelModel, llr, transmit, trial_rng
from .codes import ParityCheckMatrix, as_code, is_codeword

CSV_COLUMNS = [
    "decoder", "channel_kind", "channel_param", "rate", "n", "trials", "word_errors", "bit_errors",
    "wer", "ber", "avg_iters_all", "avg_iters_correct", "avg_iters_err", "avg_time_all_s",
    "avg_time_correct_s", "avg_time_err_s", "ml_errors", "seed",
]

ALGORITHMS = ("admm", "bp", "dual-ascent")


@dataclass(frozen=True)
class DecoderRef:
    """Decoder selection (simulator.py:53-72): ``"admm"`` and ``"bp"`` run on the GPU."""

    algo: str = "admm"
    config: AdmmConfig | BpConfig | None = None

    def __post_init__(self) -> None:
        if self.algo not in ALGORITHMS:
            raise ValueError(f"unknown decoder {self.algo!r}; use one of {ALGORITHMS}")

    def admm_config(self) -> AdmmConfig | BpConfig:
        """The decoder's config (defaults as simulator.py:64-72)."""
        if self.algo == "admm":
            return self.config if self.config is not None else AdmmConfig()
        if self.algo == "bp":
            return self.config if self.config is not None else BpConfig()
        raise NotImplementedError(
            f"decoder {self.algo!r} is a CPU baseline of the reference; 'admm' and 'bp' run on the GPU")

    def bind(self, code) -> Callable[[NDArray[np.float64]], DecodeOutput]:
        cfg = self.admm_config()
        if self.algo == "bp":
            return lambda g: decode_bp(g, code, cfg)
        return lambda g: decode(g, code, cfg)


class MlOutcome(enum.Enum):
    SUCCESS = "ml_success"
    CERTIFIED_ERROR = "ml_certified_error"
    UNKNOWN_AS_SUCCESS = "unknown_counted_as_success"


def ml_account(output: DecodeOutput, gamma, code, transmitted: ArrayLike | None = None) -> MlOutcome:
    """ML lower-bound accounting of one word error (simulator.py:83-106)."""
    code = as_code(code)
    sent = np.zeros(code.n_vars, np.uint8) if transmitted is None else np.asarray(transmitted, np.uint8)
    est = output.hard_decision
    if not is_codeword(code, est):
        return MlOutcome.UNKNOWN_AS_SUCCESS
    g = np.asarray(gamma, dtype=float)
    if float(g @ est) < float(g @ sent):
        return MlOutcome.CERTIFIED_ERROR
    return MlOutcome.SUCCESS


@dataclass
class TrialStats:
    """Accumulated statistics of one (decoder, channel point) run (simulator.py:109-153)."""

    decoder_id: str
    channel_kind: str
    channel_param: float
    seed: int
    n_vars: int
    rate: float
    trials: int = 0
    word_errors: int = 0
    bit_errors: int = 0
    iter_sum_correct: int = 0
    iter_sum_erroneous: int = 0
    time_sum_correct: float = 0.0
    time_sum_erroneous: float = 0.0
    ml_errors: int = 0

    @property
    def wer(self) -> float:
        return self.word_errors / self.trials if self.trials else 0.0

    @property
    def ber(self) -> float:
        return self.bit_errors / (self.trials * self.n_vars) if self.trials else 0.0

    def merge(self, other: "TrialStats") -> "TrialStats":
        if (self.decoder_id, self.channel_kind, self.channel_param) != (
                other.decoder_id, other.channel_kind, other.channel_param):
            raise ValueError("cannot merge stats from different runs")
        return replace(
            self,
            trials=self.trials + other.trials,
            word_errors=self.word_errors + other.word_errors,
            bit_errors=self.bit_errors + other.bit_errors,
            iter_sum_correct=self.iter_sum_correct + other.iter_sum_correct,
            iter_sum_erroneous=self.iter_sum_erroneous + other.iter_sum_erroneous,
            time_sum_correct=self.time_sum_correct + other.time_sum_correct,
            time_sum_erroneous=self.time_sum_erroneous + other.time_sum_erroneous,
            ml_errors=self.ml_errors + other.ml_errors,
        )


def _decode_wave(code, channel, cfg, sent, seed, point, trials: range, *, frames: str, dtype, device, engine):
    """Decode one contiguous block of trials; returns per-trial records as
    numpy arrays (word_error, bit_errors, iterations, seconds, ml_error)."""
    B = len(trials)
    t0 = time.perf_counter()
    all_zero = not np.any(sent)
    bp = isinstance(cfg, BpConfig)
    if frames == "device":
        if not all_zero:
            raise ValueError("frames='device' synthesises the all-zero codeword only")
        if bp:
            gam = synth_llr(code.n_vars, channel, seed=seed, point=point, trial0=trials.start, batch=B,
                            dtype=dtype, device=device)
            res = decode_bp_batch(gam, code, cfg, dtype=dtype, device=device, want_beliefs=False, want_x=False,
                                  validate=False)
        else:
            # All-zero codeword: the bit errors are the hard-decision weight and
            # cost_sent = 0, so no per-variable output is needed (the wide
            # kernel then retires frames without a retiring pass); the rare
            # certified error words get their hard decisions and LLRs from a
            # re-decode of those trials (a trial's result does not depend on
            # its batch).
            res = decode_synth(code, channel, cfg, seed=seed, point=point, trial0=trials.start, batch=B,
                               dtype=dtype, device=device, want_hard=False, engine=engine)
            bit_err = res.weight.to(torch.int64)
            word_err = bit_err > 0
            ml = torch.zeros(B, dtype=torch.bool, device=bit_err.device)
            # re-decode on the kernel that decoded the wave (a frame's result is
            # independent of its batch and slot on one kernel, but the kernels
            # round differently in fp32; batch 1 would otherwise pick the sharded one)
            eng1 = "wide" if res.info.get("kernel") == 5 else engine
            for k in (word_err & res.codeword).nonzero().flatten().tolist():
                t = trials.start + k
                one = decode_synth(code, channel, cfg, seed=seed, point=point, trial0=t, batch=1, dtype=dtype,
                                   device=device, want_hard=True, engine=eng1)
                g1 = synth_llr(code.n_vars, channel, seed=seed, point=point, trial0=t, batch=1,
                               dtype=torch.float64, device=device)
                ml[k] = bool((g1[0] * one.hard[0].to(torch.float64)).sum() < 0)  # cost_est < cost_sent = 0
            out = (word_err.cpu().numpy(), bit_err.cpu().numpy(), res.iterations.cpu().numpy().astype(np.int64),
                   ml.cpu().numpy())
            dt = time.perf_counter() - t0
            return out[0], out[1], out[2], np.full(B, dt / max(B, 1)), out[3]
    elif frames == "reference":
        gam_np = np.empty((B, code.n_vars))
        for k, t in enumerate(trials):
            gam_np[k] = llr(transmit(sent, channel, trial_rng(seed, point, t)), channel)
        gam = torch.from_numpy(gam_np).to(device)
        if bp:
            res = decode_bp_batch(gam, code, cfg, dtype=dtype, device=device, want_beliefs=False, want_x=False,
                                  validate=False)
        else:
            res = decode_batch(gam, code, cfg, dtype=dtype, device=device, want_x=False, want_hard=True,
                               validate=False, engine=engine)
    else:
        raise ValueError("frames must be 'reference' or 'device'")
    hard = res.hard
    sent_t = torch.as_tensor(sent, device=hard.device)
    bit_err = (hard != sent_t).sum(dim=1).to(torch.int64)
    word_err = bit_err > 0
    if gam is None:
        gam = synth_llr(code.n_vars, channel, seed=seed, point=point, trial0=trials.start, batch=B,
                        dtype=torch.float64, device=device)
    cost_est = (gam.to(torch.float64) * hard.to(torch.float64)).sum(dim=1)
    cost_sent = (gam.to(torch.float64) * sent_t.to(torch.float64)).sum(dim=1)
    ml = word_err & res.codeword & (cost_est < cost_sent)
    out = (word_err.cpu().numpy(), bit_err.cpu().numpy(), res.iterations.cpu().numpy().astype(np.int64),
           ml.cpu().numpy())
    dt = time.perf_counter() - t0
    return out[0], out[1], out[2], np.full(B, dt / max(B, 1)), out[3]


def run_point(code, channel: ChannelModel, decoder: DecoderRef, *, n_trials: int | None = None,
              target_errors: int | None = None, max_trials: int = 1_000_000, seed: int = 0,
              point_index: int = 0, workers: int = 1, transmitted: ArrayLike | None = None,
              pool=None, frames: str = "reference", dtype=torch.float64, device=None,
              batch_size: int = 4096, engine: str = "auto") -> TrialStats:
    """Monte-Carlo decode trials at one channel point (simulator.py:223-318).

    ``workers``/``pool`` are accepted for signature compatibility and ignored
    (the batch is the parallelism).  Results depend only on
    (seed, point_index, trial index)."""
    code = as_code(code)
    cfg = decoder.admm_config()
    if (n_trials is None) == (target_errors is None):
        raise ValueError("give exactly one of n_trials or target_errors")
    if n_trials is not None and n_trials < 1:
        raise ValueError("n_trials must be at least 1")
    if target_errors is not None and target_errors < 1:
        raise ValueError("target_errors must be at least 1")
    sent = np.zeros(code.n_vars, dtype=np.uint8) if transmitted is None else np.asarray(transmitted, np.uint8)
    if not is_codeword(code, sent):
        raise ValueError("transmitted word must be a codeword")
    dev = torch.device(device if device is not None else "cuda")

    parts = []

    def wave(lo, hi):
        parts.append(_decode_wave(code, channel, cfg, sent, seed, point_index, range(lo, hi), frames=frames,
                                  dtype=dtype, device=dev, engine=engine))

    if n_trials is not None:
        for lo in range(0, n_trials, batch_size):
            wave(lo, min(n_trials, lo + batch_size))
    else:
        errors, nxt = 0, 0
        while errors < target_errors and nxt < max_trials:
            hi = min(nxt + batch_size, max_trials)
            wave(nxt, hi)
            errors += int(parts[-1][0].sum())
            nxt = hi
    we = np.concatenate([p[0] for p in parts]) if parts else np.zeros(0, bool)
    be = np.concatenate([p[1] for p in parts]) if parts else np.zeros(0, np.int64)
    it = np.concatenate([p[2] for p in parts]) if parts else np.zeros(0, np.int64)
    tm = np.concatenate([p[3] for p in parts]) if parts else np.zeros(0)
    ml = np.concatenate([p[4] for p in parts]) if parts else np.zeros(0, bool)
    if target_errors is not None and we.sum() >= target_errors:
        # Truncate exactly at the trial that met the target (simulator.py:286-294).
        k = int(np.nonzero(np.cumsum(we) == target_errors)[0][0])
        we, be, it, tm, ml = we[: k + 1], be[: k + 1], it[: k + 1], tm[: k + 1], ml[: k + 1]

    st = TrialStats(decoder_id=decoder.algo, channel_kind=channel.kind, channel_param=channel.param,
                    seed=seed, n_vars=code.n_vars, rate=code.design_rate)
    st.trials = int(we.size)
    st.word_errors = int(we.sum())
    st.bit_errors = int(be[we].sum())
    st.iter_sum_erroneous = int(it[we].sum())
    st.iter_sum_correct = int(it[~we].sum())
    st.time_sum_erroneous = float(tm[we].sum())
    st.time_sum_correct = float(tm[~we].sum())
    st.ml_errors = int(ml[we].sum())
    return st


def sweep(code, channel_points: Sequence[ChannelModel], decoder: DecoderRef, *, n_trials: int | None = None,
          target_errors: int | None = None, max_trials: int = 1_000_000, seed: int = 0, workers: int = 1,
          **kw) -> list[TrialStats]:
    """One :func:`run_point` per channel point (simulator.py:321-352)."""
    return [run_point(code, ch, decoder, n_trials=n_trials, target_errors=target_errors, max_trials=max_trials,
                      seed=seed, point_index=k, workers=workers, **kw)
            for k, ch in enumerate(channel_points)]


def _fmt(v: float) -> str:
    return f"{v:.6g}"


def stats_to_csv(stats: Sequence[TrialStats], timing: bool = True) -> str:
    """CSV with the reference's columns and formatting (simulator.py:359-394)."""
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    w.writerow(CSV_COLUMNS)
    for s in stats:
        correct = s.trials - s.word_errors
        it_tot = s.iter_sum_correct + s.iter_sum_erroneous
        tm_tot = s.time_sum_correct + s.time_sum_erroneous
        w.writerow([
            s.decoder_id, s.channel_kind, _fmt(s.channel_param), _fmt(s.rate), s.n_vars, s.trials,
            s.word_errors, s.bit_errors, _fmt(s.wer), _fmt(s.ber),
            _fmt(it_tot / s.trials) if s.trials else "",
            _fmt(s.iter_sum_correct / correct) if correct else "",
            _fmt(s.iter_sum_erroneous / s.word_errors) if s.word_errors else "",
            _fmt(tm_tot / s.trials) if timing and s.trials else "",
            _fmt(s.time_sum_correct / correct) if timing and correct else "",
            _fmt(s.time_sum_erroneous / s.word_errors) if timing and s.word_errors else "",
            s.ml_errors, s.seed,
        ])
    return buf.getvalue()
