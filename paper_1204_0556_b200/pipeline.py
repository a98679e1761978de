"""Pipelined host-to-host decoding: the end-to-end path of the public API.

``HostPipeline.run(chunks)`` takes host LLR blocks ([B_i, N], ideally pinned)
and returns host results per block, overlapping three streams:

    copy-in  (H2D of block i+1)  |  decode (block i)  |  copy-out (D2H of block i-1)

Device buffers are allocated once (two input slots, two output slots).  With
``reuse_outputs=True`` the pinned host result buffers are allocated once per
chunk position and reused by the next ``run`` (results stay valid until
then), so the steady state allocates nothing -- pinned allocations are
synchronous and cost milliseconds each.  This is the batched counterpart of the
reference's per-trial loop ``decode_fn(gamma)`` (simulator.py:172-177),
where the host produces LLRs and consumes hard decisions.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _lib
from .admm_decoder import AdmmConfig, _dtype_code, device_graph, launch
from .codes import as_code


@dataclass
class HostResult:
    iterations: torch.Tensor  # [B] int32 (host)
    flags: torch.Tensor       # [B] uint8 (host)
    weight: torch.Tensor      # [B] int32 (host)
    hard: torch.Tensor | None  # [B, N] uint8 (host)


class HostPipeline:
    def __init__(self, code, config: AdmmConfig, *, dtype=torch.float32, device=None, max_batch: int,
                 want_hard: bool = True, reuse_outputs: bool = False):
        self.code = as_code(code)
        self.cfg = config
        self.dev = torch.device(device if device is not None else "cuda")
        self.tdt = torch.float64 if _dtype_code(dtype) == _lib.ADMM_F64 else torch.float32
        self.code_dt = _dtype_code(self.tdt)
        self.dg = device_graph(self.code, self.dev)
        self.max_batch = int(max_batch)
        self.want_hard = want_hard
        N = self.code.n_vars
        mk = lambda *s, dt: [torch.empty(s, dtype=dt, device=self.dev) for _ in range(2)]  # noqa: E731
        self.g = mk(self.max_batch, N, dt=self.tdt)
        self.iters = mk(self.max_batch, dt=torch.int32)
        self.flags = mk(self.max_batch, dt=torch.uint8)
        self.weight = mk(self.max_batch, dt=torch.int32)
        self.hard = mk(self.max_batch, N, dt=torch.uint8) if want_hard else [None, None]
        ws = self.dg.workspace_bytes(self.code_dt, self.max_batch)
        self.ws = mk(ws, dt=torch.uint8)
        self.s_in = torch.cuda.Stream(self.dev)
        self.s_out = torch.cuda.Stream(self.dev)
        self.reuse_outputs = reuse_outputs
        self._host_out: dict[tuple[int, int], HostResult] = {}

    def _host_result(self, i: int, B: int) -> HostResult:
        key = (i, B)
        if self.reuse_outputs and key in self._host_out:
            return self._host_out[key]
        res = HostResult(
            iterations=torch.empty(B, dtype=torch.int32, pin_memory=True),
            flags=torch.empty(B, dtype=torch.uint8, pin_memory=True),
            weight=torch.empty(B, dtype=torch.int32, pin_memory=True),
            hard=torch.empty((B, self.code.n_vars), dtype=torch.uint8, pin_memory=True)
            if self.want_hard else None)
        if self.reuse_outputs:
            self._host_out[key] = res
        return res

    def h2d_bytes_per_run(self, chunks) -> int:
        return sum(c.shape[0] * c.shape[1] * torch.tensor([], dtype=self.tdt).element_size() for c in chunks)

    def d2h_bytes_per_run(self, chunks) -> int:
        per = 4 + 1 + 4 + (self.code.n_vars if self.want_hard else 0)
        return sum(c.shape[0] * per for c in chunks)

    def run(self, chunks) -> list[HostResult]:
        comp = torch.cuda.current_stream(self.dev)
        self.s_in.wait_stream(comp)
        self.s_out.wait_stream(comp)
        in_ready = [torch.cuda.Event(), torch.cuda.Event()]
        slot_free = [None, None]    # decode of the slot's previous block finished
        out_done = [None, None]     # copy-out of the slot's previous block finished
        results = []
        for i, host in enumerate(chunks):
            k = i & 1
            B = host.shape[0]
            if B > self.max_batch:
                raise ValueError("chunk larger than max_batch")
            gbuf = self.g[k][:B]
            with torch.cuda.stream(self.s_in):
                if slot_free[k] is not None:
                    self.s_in.wait_event(slot_free[k])
                gbuf.copy_(host.to(self.tdt) if host.dtype != self.tdt else host, non_blocking=True)
                in_ready[k].record(self.s_in)
            comp.wait_event(in_ready[k])
            if out_done[k] is not None:
                comp.wait_event(out_done[k])
            hard = self.hard[k][:B] if self.want_hard else None
            launch(self.dg, self.code_dt, gbuf, self.cfg, self.iters[k][:B], self.flags[k][:B],
                   self.weight[k][:B], hard=hard, workspace=self.ws[k], stream=comp)
            ev = torch.cuda.Event()
            ev.record(comp)
            slot_free[k] = ev
            res = self._host_result(i, B)
            with torch.cuda.stream(self.s_out):
                self.s_out.wait_event(ev)
                res.iterations.copy_(self.iters[k][:B], non_blocking=True)
                res.flags.copy_(self.flags[k][:B], non_blocking=True)
                res.weight.copy_(self.weight[k][:B], non_blocking=True)
                if self.want_hard:
                    res.hard.copy_(hard, non_blocking=True)
                od = torch.cuda.Event()
                od.record(self.s_out)
                out_done[k] = od
            results.append(res)
        comp.wait_stream(self.s_out)
        comp.wait_stream(self.s_in)
        return results
