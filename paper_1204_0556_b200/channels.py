"""Binary symmetric and binary-input AWGN channels (host side).

Mirror of ``/root/reference/pkg/src/polylp/channels.py``: same dataclasses,
validation, negative-LLR convention (positive favours bit 0) and seeded
sampling, so frames built here are bit-identical to the reference's.  The
per-trial seeding recipe of the reference harness
(``SeedSequence(entropy=seed, spawn_key=(point, trial))``,
simulator.py:169-173) is exposed as :func:`trial_gamma` /
:func:`trial_gammas`; that is how parity inputs are made.

Device-side synthesis for throughput runs (Philox, statistically equivalent,
not bit-identical) lives in :func:`awgn_gammas_device`.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Union

import numpy as np
from numpy.typing import ArrayLike, NDArray


@dataclass(frozen=True)
class Bsc:
    """Binary symmetric channel, crossover p in (0, 0.5] (channels.py:19-33)."""

    p: float

    def __post_init__(self) -> None:
        if not (0.0 < self.p <= 0.5):
            raise ValueError("BSC crossover probability must be in (0, 0.5]")

    kind = "bsc"

    @property
    def param(self) -> float:
        return self.p


@dataclass(frozen=True)
class Awgn:
    """BPSK over AWGN at Eb/N0 ``snr_db`` for a rate-``rate`` code (channels.py:36-61)."""

    snr_db: float
    rate: float

    def __post_init__(self) -> None:
        if not (0.0 < self.rate <= 1.0):
            raise ValueError("code rate must be in (0, 1]")
        if not math.isfinite(self.snr_db):
            raise ValueError("snr_db must be finite")

    kind = "awgn"

    @property
    def param(self) -> float:
        return self.snr_db

    @property
    def noise_variance(self) -> float:
        return 1.0 / (2.0 * self.rate * 10.0 ** (self.snr_db / 10.0))


ChannelModel = Union[Bsc, Awgn]


def transmit(x: ArrayLike, ch: ChannelModel, seed) -> NDArray:
    """Send bits through the channel (channels.py:73-91): hard bits for the
    BSC, real samples for AWGN.  Uses exactly the reference's draws."""
    bits = np.asarray(x)
    if bits.ndim != 1:
        raise ValueError("codeword must be a 1-D bit vector")
    if not np.all((bits == 0) | (bits == 1)):
        raise ValueError("codeword entries must be 0 or 1")
    rng = seed if isinstance(seed, np.random.Generator) else np.random.default_rng(seed)
    if isinstance(ch, Bsc):
        flips = rng.random(bits.size) < ch.p
        return (bits.astype(np.uint8) ^ flips.astype(np.uint8)).astype(np.uint8)
    sym = 1.0 - 2.0 * bits.astype(float)
    return sym + math.sqrt(ch.noise_variance) * rng.standard_normal(bits.size)


def llr(received: ArrayLike, ch: ChannelModel) -> NDArray[np.float64]:
    """Negative LLRs in nats (channels.py:94-110)."""
    y = np.asarray(received)
    if y.ndim != 1:
        raise ValueError("received vector must be 1-D")
    if isinstance(ch, Bsc):
        if not np.all((y == 0) | (y == 1)):
            raise ValueError("BSC received symbols must be 0 or 1")
        base = math.log((1.0 - ch.p) / ch.p)
        return (1.0 - 2.0 * y.astype(float)) * base
    return 2.0 * np.asarray(y, dtype=float) / ch.noise_variance


def trial_rng(seed: int, point: int, trial: int) -> np.random.Generator:
    """The reference harness's per-trial generator (simulator.py:169-171)."""
    return np.random.default_rng(np.random.SeedSequence(entropy=seed, spawn_key=(point, trial)))


def trial_gamma(n_vars: int, ch: ChannelModel, seed: int, point: int, trial: int,
                transmitted: ArrayLike | None = None) -> NDArray[np.float64]:
    """LLRs of one trial, bit-identical to the reference harness's frame."""
    sent = np.zeros(n_vars, dtype=np.uint8) if transmitted is None else np.asarray(transmitted, np.uint8)
    return llr(transmit(sent, ch, trial_rng(seed, point, trial)), ch)


def trial_gammas(n_vars: int, ch: ChannelModel, seed: int, point: int, trials,
                 transmitted: ArrayLike | None = None) -> NDArray[np.float64]:
    """Stack of :func:`trial_gamma` frames, shape (len(trials), n_vars)."""
    trials = list(trials)
    out = np.empty((len(trials), n_vars), dtype=np.float64)
    for k, t in enumerate(trials):
        out[k] = trial_gamma(n_vars, ch, seed, point, t, transmitted)
    return out


def awgn_gammas_device(n_frames: int, n_vars: int, snr_db: float, rate: float, *,
                       seed: int, device="cuda", dtype=None):
    """All-zero-codeword BPSK/AWGN LLRs generated on the device with torch's
    Philox generator: gamma = 2 (1 + sigma n) / sigma^2.  Statistically the
    channel of channels.py:89-91,110; not bit-identical to numpy."""
    import torch

    dtype = dtype or torch.float32
    var = Awgn(snr_db, rate).noise_variance
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    y = torch.randn((n_frames, n_vars), generator=g, device=device, dtype=torch.float32)
    y.mul_(math.sqrt(var)).add_(1.0).mul_(2.0 / var)
    return y.to(dtype)


def bsc_gammas_device(n_frames: int, n_vars: int, p: float, *, seed: int, device="cuda", dtype=None):
    """All-zero-codeword BSC LLRs on the device: +-log((1-p)/p)."""
    import torch

    dtype = dtype or torch.float32
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    flips = torch.rand((n_frames, n_vars), generator=g, device=device) < p
    base = math.log((1.0 - p) / p)
    return torch.where(flips, -base, base).to(dtype)
