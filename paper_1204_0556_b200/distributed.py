"""Frame-sharded multi-GPU decoding.

Frames are independent, so N GPUs split the trial indices of every channel
point into contiguous blocks (rank g owns ``shard(F, g, N)``); each rank
rebuilds the same Tanner graph, decodes its block, and the only cross-GPU
traffic is ONE all-reduce of int64 counters -- the ``TrialStats`` fields of
the reference harness (simulator.py:109-126, merge semantics :136-153) plus
converged frames and edge-updates.

Because every frame's LLRs derive from (seed, point, trial)
(simulator.py:169-171), the merged statistics do not depend on the number of
ranks -- the GPU analogue of the reference's worker invariance
(tests/test_acceptance.py:305-320).  ``tests/test_distributed.py`` checks
that with the gloo backend at world size 2.
"""

from __future__ import annotations

from typing import Callable

import numpy as np
import torch
import torch.distributed as dist

#: Counter layout of one channel point (int64).
COUNTERS = ("trials", "word_errors", "bit_errors", "iter_sum_correct", "iter_sum_erroneous",
            "ml_errors", "converged", "edge_updates")


def shard(n_trials: int, rank: int, world: int) -> range:
    """Contiguous block of trial indices owned by ``rank`` (sizes differ by <= 1)."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    base, extra = divmod(n_trials, world)
    lo = rank * base + min(rank, extra)
    return range(lo, lo + base + (1 if rank < extra else 0))


def counters_from_results(iterations, weight, converged, codeword, cost, n_edges: int) -> torch.Tensor:
    """Per-point counters from per-frame decode results (all-zero codeword sent).

    word error  <=> Hamming weight of the hard decision > 0     (simulator.py:177-178)
    ML error    <=> word error, hard decision is a codeword and its cost
                    gamma . x_hat < gamma . 0 = 0                 (simulator.py:83-106)
    """
    it = torch.as_tensor(iterations).to(torch.int64)
    w = torch.as_tensor(weight).to(torch.int64)
    conv = torch.as_tensor(converged).to(torch.bool)
    cw = torch.as_tensor(codeword).to(torch.bool)
    cost = torch.as_tensor(cost).to(torch.float64)
    err = w > 0
    zero = torch.zeros((), dtype=torch.int64, device=it.device)
    return torch.stack([
        torch.tensor(it.numel(), dtype=torch.int64, device=it.device),
        err.sum(),
        w.sum(),
        torch.where(err, zero, it).sum(),
        torch.where(err, it, zero).sum(),
        (err & cw & (cost < 0)).sum(),
        conv.sum(),
        it.sum() * int(n_edges),
    ])


def allreduce_counters(c: torch.Tensor, group=None) -> torch.Tensor:
    """Sum counters over all ranks (one collective; no-op when not initialised)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(c, op=dist.ReduceOp.SUM, group=group)
    return c


def max_over_ranks(x: float, device=None, group=None) -> float:
    """Max of a per-rank scalar (used for device-timed elapsed seconds)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        t = torch.tensor([float(x)], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
        return float(t.item())
    return float(x)


def counters_as_dict(c: torch.Tensor) -> dict:
    return dict(zip(COUNTERS, [int(v) for v in c.cpu().tolist()]))


def gpu_decode_fn(code, config, *, dtype=torch.float64, device=None) -> Callable:
    """Default per-shard decoder: the sm_100a kernels through decode_batch.
    Returns (iterations, weight, converged, codeword, cost) for a [B, N] block."""
    from .admm_decoder import decode_batch

    def run(gammas: np.ndarray):
        g = torch.as_tensor(gammas, dtype=torch.float64, device=device or "cuda")
        res = decode_batch(g, code, config, dtype=dtype, want_x=False, want_hard=True)
        cost = (g * res.hard.to(torch.float64)).sum(dim=1)
        return res.iterations, res.weight, res.converged, res.codeword, cost

    return run


def run_point_sharded(code, gamma_of_trial: Callable[[int], np.ndarray], n_trials: int, *,
                      decode_fn: Callable, rank: int = 0, world: int = 1, chunk: int = 4096,
                      group=None, device="cpu") -> dict:
    """Decode this rank's shard of ``n_trials`` frames and merge the counters
    of all ranks with one all-reduce.  ``gamma_of_trial(t)`` must be a pure
    function of the trial index (seeded like simulator.py:169-173)."""
    mine = shard(n_trials, rank, world)
    total = torch.zeros(len(COUNTERS), dtype=torch.int64, device=device)
    for lo in range(mine.start, mine.stop, chunk):
        idx = range(lo, min(lo + chunk, mine.stop))
        gam = np.stack([gamma_of_trial(t) for t in idx])
        it, w, conv, cw, cost = decode_fn(gam)
        total += counters_from_results(it, w, conv, cw, cost, code.n_edges).to(device)
    return counters_as_dict(allreduce_counters(total, group))
