"""ADMM-LP decoder: the reference-compatible API over the sm_100a kernels.

Mirror of ``polylp.admm_decoder`` (/root/reference/pkg/src/polylp/admm_decoder.py):

* :class:`AdmmConfig` -- same fields, defaults and validation (:27-44);
* :class:`DecodeOutput` and the ``STATUS_*`` strings (:23-24, :74-89),
  :func:`make_output` (:92-105);
* :class:`AdmmState` and the step functions :func:`x_update`,
  :func:`z_update`, :func:`lambda_update` (:47-71, :108-149) -- the same
  state object driven by hand, each step one batched sm_100a kernel
  (csrc/steps.cu);
* :func:`decode` ``(gamma, code, config) -> DecodeOutput`` -- same
  arguments, errors and output convention (:152-182), computed in fp64 on the
  GPU (the parity mode);

and the B200 batch entry point :func:`decode_batch`, which decodes a
``[B, N]`` block of frames in one launch (fp32 throughput mode or fp64
parity mode) and returns per-frame results as device tensors.

There is no CPU fallback: a missing extension raises ``RuntimeError``.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch
from numpy.typing import ArrayLike, NDArray

from . import _lib
from .codes import ParityCheckMatrix, as_code

INTEGRALITY_TOL = 1e-5
STATUS_CONVERGED = "Converged"
STATUS_MAX_ITERS = "MaxIters"


@dataclass(frozen=True)
class AdmmConfig:
    """Penalty, stopping tolerance, iteration cap and over-relaxation
    (admm_decoder.py:27-44)."""

    mu: float = 3.0
    epsilon: float = 1e-5
    t_max: int = 1000
    rho: float = 1.9

    def __post_init__(self) -> None:
        if self.mu <= 0:
            raise ValueError("mu must be positive")
        if self.epsilon <= 0:
            raise ValueError("epsilon must be positive")
        if self.t_max < 1:
            raise ValueError("t_max must be at least 1")
        if not (1.0 <= self.rho < 2.0):
            raise ValueError("rho must be in [1, 2)")


@dataclass(frozen=True)
class DecodeOutput:
    """Result of one decode (admm_decoder.py:74-89)."""

    x: NDArray[np.float64]
    status: str
    integral: bool
    iterations: int
    hard_decision: NDArray[np.uint8]
    ml_certificate: bool


def make_output(x, status: str, iterations: int, code) -> DecodeOutput:
    """Hard decision, integrality and ML certificate of a final iterate
    (admm_decoder.py:92-105); host arrays, as the reference."""
    from .codes import is_codeword

    x = np.asarray(x, dtype=float)
    hard = (x > 0.5).astype(np.uint8)
    integral = bool(np.all(np.minimum(np.abs(x), np.abs(1.0 - x)) <= INTEGRALITY_TOL))
    cert = integral and is_codeword(as_code(code), hard)
    return DecodeOutput(x=x, status=status, integral=integral, iterations=iterations, hard_decision=hard,
                        ml_certificate=cert)


@dataclass
class AdmmState:
    """Iterates of a decode (admm_decoder.py:47-71): variables ``x`` (N),
    replicas ``z``, duals ``lam``, previous replicas ``z_prev`` and the
    over-relaxed mixture ``w`` (E, edge-flat in check order; the slice of
    check j is ``code.check_slice(j)``).

    As in the reference the fields are host numpy arrays of one frame; the
    step functions then run in fp64.  They may also be CUDA tensors, one
    frame ([N] / [E]) or a batch ([B, N] / [B, E]), float32 or float64:
    the steps then stay on the device in that dtype.
    """

    x: NDArray[np.float64] | torch.Tensor
    z: NDArray[np.float64] | torch.Tensor
    lam: NDArray[np.float64] | torch.Tensor
    z_prev: NDArray[np.float64] | torch.Tensor
    w: NDArray[np.float64] | torch.Tensor = field(default_factory=lambda: np.empty(0))
    iterations: int = 0

    @classmethod
    def initial(cls, code, *, batch: int | None = None, dtype=None, device=None) -> "AdmmState":
        """Zero state (admm_decoder.py:63-71).  With ``device`` (or ``batch``)
        the state is a CUDA tensor state of ``batch`` frames."""
        code = as_code(code)
        e = code.n_edges
        if device is None and batch is None:
            return cls(x=np.zeros(code.n_vars), z=np.zeros(e), lam=np.zeros(e), z_prev=np.zeros(e))
        dev = torch.device(device if device is not None else "cuda")
        tdt = torch.float64 if dtype is None or _dtype_code(dtype) == _lib.ADMM_F64 else torch.float32
        shp = (() if batch is None else (int(batch),))
        zeros = lambda n: torch.zeros(shp + (n,), dtype=tdt, device=dev)  # noqa: E731
        return cls(x=zeros(code.n_vars), z=zeros(e), lam=zeros(e), z_prev=zeros(e), w=zeros(e))


class _StepIO:
    """Host <-> device marshalling of one step: numpy in -> fp64 CUDA rows ->
    numpy out, or CUDA tensors in -> CUDA tensors out (same dtype/shape)."""

    def __init__(self, state: AdmmState, code):
        self.code = as_code(code)
        ref = state.z
        self.host = not (isinstance(ref, torch.Tensor) and ref.is_cuda)
        if self.host:
            self.dev = torch.device("cuda", torch.cuda.current_device())
            self.tdt = torch.float64
            self.batched = np.ndim(ref) == 2
        else:
            self.dev = ref.device
            self.tdt = ref.dtype
            self.batched = ref.ndim == 2
        self.dt_code = _dtype_code(self.tdt)
        self.dg = device_graph(self.code, self.dev)
        self.stream = torch.cuda.current_stream(self.dev)

    def rows(self, a, n: int) -> torch.Tensor:
        t = torch.as_tensor(a).to(device=self.dev, dtype=self.tdt)
        if t.shape[-1] != n:
            raise ValueError(f"expected trailing dimension {n}, got {tuple(t.shape)}")
        return t.reshape(-1, n).contiguous()

    def out(self, t: torch.Tensor):
        t = t if self.batched else t[0]
        return t.cpu().numpy() if self.host else t


def x_update(state: AdmmState, code, gamma, config: AdmmConfig):
    """Average the dual-adjusted replicas, step against the LLRs, clamp
    (admm_decoder.py:108-124): one sm_100a kernel (admm_x_update)."""
    io = _StepIO(state, code)
    N, E = io.code.n_vars, io.code.n_edges
    z, lam, g = io.rows(state.z, E), io.rows(state.lam, E), io.rows(gamma, N)
    B = z.shape[0]
    if g.shape[0] != B:
        g = g.expand(B, N).contiguous()
    x = torch.empty((B, N), dtype=io.tdt, device=io.dev)
    _lib.check(_lib.load().admm_x_update(io.dg.handle, io.dt_code, B, z.data_ptr(), lam.data_ptr(), E, g.data_ptr(),
                                         N, float(config.mu), x.data_ptr(), N, io.stream.cuda_stream))
    state.x = io.out(x)
    return state.x


def z_update(state: AdmmState, code, config: AdmmConfig):
    """Project each check's over-relaxed replica target onto the parity
    polytope (admm_decoder.py:127-141): one kernel (admm_z_update).
    Sets ``z_prev``, ``w`` and ``z`` as the reference does."""
    io = _StepIO(state, code)
    N, E = io.code.n_vars, io.code.n_edges
    x, z, lam = io.rows(state.x, N), io.rows(state.z, E), io.rows(state.lam, E)
    B = z.shape[0]
    z_new = torch.empty((B, E), dtype=io.tdt, device=io.dev)
    w = torch.empty((B, E), dtype=io.tdt, device=io.dev)
    _lib.check(_lib.load().admm_z_update(io.dg.handle, io.dt_code, B, x.data_ptr(), N, z.data_ptr(), lam.data_ptr(),
                                         E, float(config.mu), float(config.rho), z_new.data_ptr(), w.data_ptr(),
                                         io.stream.cuda_stream))
    state.z_prev = state.z
    state.w = io.out(w)
    state.z = io.out(z_new)
    return state.z


def lambda_update(state: AdmmState, code, config: AdmmConfig):
    """Dual step against the residual of the same mixture the replicas saw
    (admm_decoder.py:144-149): one kernel (admm_lambda_update)."""
    io = _StepIO(state, code)
    E = io.code.n_edges
    lam, w, z = io.rows(state.lam, E), io.rows(state.w, E), io.rows(state.z, E)
    B = lam.shape[0]
    out = torch.empty((B, E), dtype=io.tdt, device=io.dev)
    _lib.check(_lib.load().admm_lambda_update(io.dg.handle, io.dt_code, B, lam.data_ptr(), w.data_ptr(), z.data_ptr(),
                                              E, float(config.mu), out.data_ptr(), io.stream.cuda_stream))
    state.lam = io.out(out)
    return state.lam


# ---------------------------------------------------------------------------
# Device graph
# ---------------------------------------------------------------------------
class DeviceGraph:
    """Owner of an ``admm_graph`` handle (immutable, one per code and device)."""

    def __init__(self, code: ParityCheckMatrix, device: int, engine: str = "auto"):
        lib = _lib.load()
        self.code = code
        self.device = int(device)
        self.engine = engine
        ptr = np.ascontiguousarray(code.check_ptr, dtype=np.int32)
        ev = np.ascontiguousarray(code.edge_var, dtype=np.int32)
        h = ctypes.c_void_p()
        if engine not in _lib.ENGINES:
            raise ValueError(f"unknown engine {engine!r}; use one of {sorted(_lib.ENGINES)}")
        _lib.check(lib.admm_graph_create_ex(self.device, code.n_vars, code.n_checks, ptr.ctypes.data,
                                            ev.ctypes.data, _lib.ENGINES[engine], ctypes.byref(h)))
        self._h = h
        info = _lib.GraphInfo()
        _lib.check(lib.admm_graph_get_info(self._h, ctypes.byref(info)))
        self.info = info.as_dict()

    @property
    def handle(self) -> ctypes.c_void_p:
        return self._h

    def workspace_bytes(self, dtype_code: int, batch: int) -> int:
        return int(_lib.load().admm_workspace_bytes(self._h, dtype_code, batch))

    def call_info(self, dtype_code: int, batch: int) -> dict:
        """Graph info plus the kernel a call with ``batch`` frames runs
        (``kernel``: admm_decode_kernel id, ``kernel_name``)."""
        k = int(_lib.load().admm_decode_kernel(self._h, dtype_code, batch))
        return dict(self.info, kernel=k, kernel_name=_lib.KERNELS.get(k, "?"))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                _lib.load().admm_graph_destroy(h)
            except Exception:
                pass
            self._h = None


def device_graph(code, device=None, engine: str = "auto") -> DeviceGraph:
    """The (cached) device-resident graph of ``code`` on ``device``.

    ``engine``: "auto" (resident when the code fits one SM, else streaming),
    "resident", "streaming" (codes beyond one SM: the sharded kernel below
    1024 frames per call, the wide HBM-streaming kernel from there on --
    csrc/sharded.cuh, csrc/wide.cuh), "wide" (the wide kernel for every
    batch)."""
    code = as_code(code)
    dev = torch.device(device if device is not None else "cuda")
    idx = dev.index if dev.index is not None else torch.cuda.current_device()
    key = (idx, engine)
    g = code._device_graphs.get(key)
    if g is None:
        g = DeviceGraph(code, idx, engine)
        code._device_graphs[key] = g
    return g


def _dtype_code(dtype) -> int:
    if dtype in (torch.float32, "f32", "float32", np.float32):
        return _lib.ADMM_F32
    if dtype in (torch.float64, "f64", "float64", np.float64, float):
        return _lib.ADMM_F64
    raise ValueError(f"unsupported dtype {dtype!r}; use float32 or float64")


# ---------------------------------------------------------------------------
# Batch decode
# ---------------------------------------------------------------------------
@dataclass
class BatchResult:
    """Per-frame results of :func:`decode_batch` (device tensors)."""

    iterations: torch.Tensor          # [B] int32
    flags: torch.Tensor               # [B] uint8, ADMM_FLAG_* bits
    weight: torch.Tensor              # [B] int32, Hamming weight of the hard decision
    x: torch.Tensor | None = None     # [B, N] final x
    hard: torch.Tensor | None = None  # [B, N] uint8
    z: torch.Tensor | None = None     # [B, E] final replicas (reference edge order)
    lam: torch.Tensor | None = None   # [B, E] final duals
    info: dict = field(default_factory=dict)

    @property
    def converged(self) -> torch.Tensor:
        return (self.flags & _lib.ADMM_FLAG_CONVERGED) != 0

    @property
    def integral(self) -> torch.Tensor:
        return (self.flags & _lib.ADMM_FLAG_INTEGRAL) != 0

    @property
    def codeword(self) -> torch.Tensor:
        return (self.flags & _lib.ADMM_FLAG_CODEWORD) != 0

    @property
    def ml_certificate(self) -> torch.Tensor:
        return self.integral & self.codeword

    def output(self, k: int) -> DecodeOutput:
        """Frame k as a reference :class:`DecodeOutput` (host arrays)."""
        if self.x is None:
            raise ValueError("decode_batch was called with want_x=False")
        x = self.x[k].detach().double().cpu().numpy()
        hard = (x > 0.5).astype(np.uint8)
        flags = int(self.flags[k])
        integral = bool(flags & _lib.ADMM_FLAG_INTEGRAL)
        return DecodeOutput(
            x=x,
            status=STATUS_CONVERGED if flags & _lib.ADMM_FLAG_CONVERGED else STATUS_MAX_ITERS,
            integral=integral,
            iterations=int(self.iterations[k]),
            hard_decision=hard,
            ml_certificate=integral and bool(flags & _lib.ADMM_FLAG_CODEWORD),
        )


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def launch(dg: DeviceGraph, code_dt: int, g: torch.Tensor, config: AdmmConfig, iters, flags, weight, *,
           x=None, hard=None, z0=None, lam0=None, z_out=None, lam_out=None, workspace, stream) -> None:
    """Enqueue one ``admm_decode_batch`` on caller-owned device buffers (no
    allocation, no validation beyond the C ABI's)."""
    N, E = dg.code.n_vars, dg.code.n_edges
    if g.shape[0] == 0:
        return
    if g.stride(1) != 1:
        raise ValueError("LLR rows must be contiguous")
    ld = g.stride(0) if g.shape[0] > 1 else N  # a single row may carry any stride(0)
    _lib.check(_lib.load().admm_decode_batch(
        dg.handle, code_dt, g.shape[0], g.data_ptr(), ld,
        float(config.mu), float(config.epsilon), int(config.t_max), float(config.rho),
        _ptr(x), N if x is None else x.stride(0), _ptr(hard), N if hard is None else hard.stride(0),
        iters.data_ptr(), flags.data_ptr(), weight.data_ptr(),
        _ptr(z0), _ptr(lam0), _ptr(z_out), _ptr(lam_out), E,
        workspace.data_ptr(), workspace.numel(), stream.cuda_stream))


def decode_batch(
    gammas,
    code,
    config: AdmmConfig = AdmmConfig(),
    *,
    dtype=torch.float64,
    device=None,
    want_x: bool = True,
    want_hard: bool = False,
    z0=None,
    lam0=None,
    want_state: bool = False,
    validate: bool = True,
    stream: torch.cuda.Stream | None = None,
    engine: str = "auto",
) -> BatchResult:
    """Decode ``gammas`` ([B, N], one frame per row) on the GPU.

    Frames are independent; the result for a frame does not depend on the
    batch it was decoded in.  ``dtype`` selects the arithmetic: float64 is
    the parity mode, float32 the throughput mode.  ``z0``/``lam0`` ([B, E],
    reference edge order) replace the zero initial state; ``want_state``
    returns the final replicas and duals.  Work is enqueued on ``stream``
    (default: the current stream) and the call does not synchronise.
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
    if z0 is not None or lam0 is not None:
        if z0 is None or lam0 is None:
            raise ValueError("z0 and lam0 go together")
    B, N, E = g.shape[0], code.n_vars, code.n_edges
    dg = device_graph(code, dev, engine)
    code_dt = _dtype_code(tdt)
    # Everything below is enqueued on `st`: the conversions, the allocations
    # (the caching allocator then ties the buffers to `st`) and the kernel.
    # `st` first waits for the caller's current stream, which produced the
    # inputs; a caller-side input tensor read on a side stream is recorded
    # on it so its memory is not reused before the kernel has read it.
    cur = torch.cuda.current_stream(dev)
    st = stream if stream is not None else cur
    if st != cur:
        st.wait_stream(cur)
        for t in (g, z0, lam0):
            if isinstance(t, torch.Tensor) and t.is_cuda:
                t.record_stream(st)
    with torch.cuda.stream(st):
        g = g.to(device=dev, dtype=tdt, non_blocking=True)
        if not g.is_contiguous() or (g.shape[0] > 1 and g.stride(0) != g.shape[1]):
            g = g.contiguous()
        if validate and not bool(torch.isfinite(g).all()):
            raise ValueError("LLR vector must be finite")
        iters = torch.empty(B, dtype=torch.int32, device=dev)
        flags = torch.empty(B, dtype=torch.uint8, device=dev)
        weight = torch.empty(B, dtype=torch.int32, device=dev)
        x = torch.empty((B, N), dtype=tdt, device=dev) if want_x else None
        hard = torch.empty((B, N), dtype=torch.uint8, device=dev) if want_hard else None
        zi = li = None
        if z0 is not None:
            zi = torch.as_tensor(z0).to(device=dev, dtype=tdt).reshape(B, E).contiguous()
            li = torch.as_tensor(lam0).to(device=dev, dtype=tdt).reshape(B, E).contiguous()
        zo = torch.empty((B, E), dtype=tdt, device=dev) if want_state else None
        lo = torch.empty((B, E), dtype=tdt, device=dev) if want_state else None
        ws_bytes = dg.workspace_bytes(code_dt, B)
        ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
        launch(dg, code_dt, g, config, iters, flags, weight, x=x, hard=hard, z0=zi, lam0=li, z_out=zo,
               lam_out=lo, workspace=ws, stream=st)
    res = BatchResult(iterations=iters, flags=flags, weight=weight, x=x, hard=hard, z=zo, lam=lo,
                      info=dg.call_info(code_dt, B))
    # the temporaries (converted inputs, workspace: up to 12 GiB on the wide
    # kernel) were allocated on `st`, so the allocator reuses their memory only
    # for work ordered after the kernel: nothing has to be kept alive
    return res


# ---------------------------------------------------------------------------
# Reference-compatible single-frame entry point
# ---------------------------------------------------------------------------
def decode(gamma: ArrayLike, code, config: AdmmConfig = AdmmConfig()) -> DecodeOutput:
    """Solve the decoding LP for one LLR vector (admm_decoder.py:152-182).

    Drop-in for ``polylp.decode``: same arguments, ``ValueError`` on a wrong
    shape or non-finite input, fp64 arithmetic, fresh output arrays.
    """
    code = as_code(code)
    gamma = np.asarray(gamma, dtype=float)
    if gamma.shape != (code.n_vars,):
        raise ValueError(f"expected a length-{code.n_vars} LLR vector")
    if not np.all(np.isfinite(gamma)):
        raise ValueError("LLR vector must be finite")
    res = decode_batch(gamma[None, :], code, config, dtype=torch.float64, validate=False)
    torch.cuda.current_stream().synchronize()
    return res.output(0)


def run_iterations(gamma, code, config: AdmmConfig, iterations: int, z0=None, lam0=None):
    """Run exactly ``iterations`` ADMM iterations (x-, z-, lambda-update, as
    admm_decoder.py:171-177) from the given replicas/duals (zeros by
    default) and return ``(x, z, lam)`` as fp64 host arrays.  The GPU
    analogue of driving ``x_update``/``z_update``/``lambda_update`` by hand
    (tests/test_admm.py:151-160 of the reference)."""
    code = as_code(code)
    cfg = AdmmConfig(mu=config.mu, epsilon=1e-300, t_max=int(iterations), rho=config.rho)
    g = np.asarray(gamma, dtype=float).reshape(1, -1)
    E = code.n_edges
    z0 = np.zeros(E) if z0 is None else np.asarray(z0, dtype=float)
    lam0 = np.zeros(E) if lam0 is None else np.asarray(lam0, dtype=float)
    if device_graph(code).info["engine"] == 3:
        # codes beyond one SM: the streaming engines keep their state in their
        # own layouts, so the iterations run as step kernels (csrc/steps.cu)
        st = AdmmState(x=np.zeros(code.n_vars), z=z0.copy(), lam=lam0.copy(), z_prev=z0.copy())
        for _ in range(int(iterations)):
            x_update(st, code, g[0], cfg)
            z_update(st, code, cfg)
            lambda_update(st, code, cfg)
        return st.x, st.z, st.lam
    res = decode_batch(g, code, cfg, dtype=torch.float64, z0=z0[None], lam0=lam0[None], want_state=True)
    torch.cuda.current_stream().synchronize()
    return (res.x[0].cpu().numpy(), res.z[0].cpu().numpy(), res.lam[0].cpu().numpy())


# ---------------------------------------------------------------------------
# Fused on-GPU frame synthesis (csrc/synth.cuh)
# ---------------------------------------------------------------------------
def _channel_struct(channel) -> "_lib.Channel":
    from .channels import Awgn, Bsc

    if isinstance(channel, Bsc):
        return _lib.Channel(1, float(channel.p), 0.0, 0.0)
    if isinstance(channel, Awgn):
        return _lib.Channel(2, 0.0, float(channel.snr_db), float(channel.rate))
    raise TypeError("channel must be a Bsc or Awgn")


def synth_llr(n_vars: int, channel, *, seed: int, point: int, trial0: int, batch: int,
              dtype=torch.float64, device=None, stream=None) -> torch.Tensor:
    """LLRs of trials trial0 .. trial0+batch-1 at channel point ``point``,
    generated on the GPU from (seed, point, trial) -- exactly the frames
    :func:`decode_synth` decodes.  All-zero codeword."""
    dev = torch.device(device if device is not None else "cuda")
    tdt = torch.float64 if _dtype_code(dtype) == _lib.ADMM_F64 else torch.float32
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    with torch.cuda.stream(st):
        out = torch.empty((batch, n_vars), dtype=tdt, device=dev)
    ch = _channel_struct(channel)
    _lib.check(_lib.load().admm_synth_llr(_dtype_code(tdt), batch, n_vars, ctypes.byref(ch), int(seed) & (2**64 - 1),
                                          int(point), int(trial0), out.data_ptr(), n_vars, st.cuda_stream))
    return out


def decode_synth(code, channel, config: AdmmConfig = AdmmConfig(), *, seed: int, point: int = 0,
                 trial0: int = 0, batch: int, dtype=torch.float32, device=None, want_x: bool = False,
                 want_hard: bool = False, engine: str = "auto", stream=None) -> BatchResult:
    """Decode trials trial0 .. trial0+batch-1 with LLRs synthesised inside
    the decode kernel (no LLR traffic).  A trial's frame depends only on
    (seed, point, trial), so results are independent of batching, engine and
    GPU count."""
    code = as_code(code)
    dev = torch.device(device if device is not None else "cuda")
    tdt = torch.float64 if _dtype_code(dtype) == _lib.ADMM_F64 else torch.float32
    dg = device_graph(code, dev, engine)
    code_dt = _dtype_code(tdt)
    B, N = int(batch), code.n_vars
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    with torch.cuda.stream(st):  # allocations tied to the stream the kernel runs on
        iters = torch.empty(B, dtype=torch.int32, device=dev)
        flags = torch.empty(B, dtype=torch.uint8, device=dev)
        weight = torch.empty(B, dtype=torch.int32, device=dev)
        x = torch.empty((B, N), dtype=tdt, device=dev) if want_x else None
        hard = torch.empty((B, N), dtype=torch.uint8, device=dev) if want_hard else None
        ws_bytes = dg.workspace_bytes(code_dt, B)
        ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=dev)
    ch = _channel_struct(channel)
    if B > 0:
        _lib.check(_lib.load().admm_decode_synth(
            dg.handle, code_dt, B, ctypes.byref(ch), int(seed) & (2**64 - 1), int(point), int(trial0),
            float(config.mu), float(config.epsilon), int(config.t_max), float(config.rho),
            _ptr(x), N, _ptr(hard), N, iters.data_ptr(), flags.data_ptr(), weight.data_ptr(),
            ws.data_ptr(), ws_bytes, st.cuda_stream))
    res = BatchResult(iterations=iters, flags=flags, weight=weight, x=x, hard=hard, info=dg.call_info(code_dt, batch))
    # (ws was allocated on `st`: its memory is only reused by work ordered after the kernel)
    return res
