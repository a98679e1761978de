"""CPU oracle for the ADMM-LP decoding hot path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference algorithm
(``polylp``, /root/reference/pkg/src/polylp).  It is the *checker* for the
CUDA path and the CPU baseline timed by ``bench.py``; nothing in the product
package imports it.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``) may use it.

Pinning: ``tests/test_oracle.py`` checks every function here against the
golden vectors in ``tests/golden/`` -- outputs of the reference package
itself, produced in the build container by ``tests/golden/make_golden.py``
(which imports the read-only reference) -- and against the reference's own
known-answer tests (test_parity_polytope.py:139-182, test_admm.py:26-135).

Each function cites the reference lines it restates.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass

import numpy as np

# parity_polytope.py:19 -- absolute tolerance on the constituent-parity test.
PARITY_TOL = 1e-9
# admm_decoder.py:21 -- integrality tolerance of the output.
INTEGRALITY_TOL = 1e-5
STATUS_CONVERGED = "Converged"
STATUS_MAX_ITERS = "MaxIters"


@dataclass(frozen=True)
class Params:
    """Decoder parameters with the reference's validation (admm_decoder.py:27-44)."""

    mu: float = 3.0
    epsilon: float = 1e-5
    t_max: int = 1000
    rho: float = 1.9

    def __post_init__(self):
        if self.mu <= 0:
            raise ValueError("mu must be positive")
        if self.epsilon <= 0:
            raise ValueError("epsilon must be positive")
        if self.t_max < 1:
            raise ValueError("t_max must be at least 1")
        if not (1.0 <= self.rho < 2.0):
            raise ValueError("rho must be in [1, 2)")


class Graph:
    """Edge-flat Tanner graph (codes.py:79-115): edges grouped by check, each
    check's variables sorted ascending."""

    def __init__(self, n_vars: int, checks):
        self.n_vars = int(n_vars)
        self.checks = [np.sort(np.asarray(c, dtype=np.int64)) for c in checks]
        self.n_checks = len(self.checks)
        self.check_deg = np.array([c.size for c in self.checks], dtype=np.int64)
        self.check_ptr = np.concatenate([[0], np.cumsum(self.check_deg)]).astype(np.int64)
        self.edge_var = np.concatenate(self.checks).astype(np.int64)
        self.n_edges = int(self.check_ptr[-1])
        self.var_deg = np.bincount(self.edge_var, minlength=self.n_vars).astype(np.int64)
        self.edge_check = np.repeat(np.arange(self.n_checks), self.check_deg)
        # one (m_d, d) edge-index block per distinct check degree
        self.blocks = {}
        for d in np.unique(self.check_deg):
            js = np.nonzero(self.check_deg == d)[0]
            self.blocks[int(d)] = self.check_ptr[js][:, None] + np.arange(int(d))[None, :]

    @classmethod
    def of(cls, code) -> "Graph":
        return cls(code.n_vars, [np.asarray(c) for c in code.check_neighborhoods])


# ---------------------------------------------------------------------------
# Parity-polytope projection (parity_polytope.py:352-421)
# ---------------------------------------------------------------------------
def project_rows(values) -> np.ndarray:
    """Row-wise Euclidean projection onto the parity polytope PP_d.

    Restates ``project_batch`` (parity_polytope.py:352-421): order each row
    descending (stable), take r = even floor of the l1 norm of the cube clip,
    test the f_r facet with tolerance PARITY_TOL (:370-382), and otherwise
    locate the shift beta on the piecewise-linear line value by evaluating it
    at every kink in [0, beta_max] and interpolating on the crossing segment
    (:385-414).
    """
    a = np.asarray(values, dtype=float)
    if a.ndim != 2 or a.shape[1] == 0:
        raise ValueError("project_batch expects an (m, d) array with d >= 1")
    if not np.all(np.isfinite(a)):
        raise ValueError("projection input must be finite")
    m, d = a.shape
    idx = np.arange(m)
    perm = np.argsort(-a, axis=1, kind="stable")
    v = a[idx[:, None], perm]                          # descending rows
    cube = np.clip(v, 0.0, 1.0)
    l1 = cube.sum(axis=1)
    r = np.minimum((2.0 * np.floor(l1 / 2.0)).astype(np.int64), d)
    last_up = np.minimum(r, d - 1)                    # last +1 position of f_r
    f = np.where(np.arange(d)[None, :] <= last_up[:, None], 1.0, -1.0)
    f_dot = 2.0 * np.cumsum(cube, axis=1)[idx, last_up] - l1
    v_up = v[idx, last_up]
    v_dn = v[idx, np.minimum(r + 1, d - 1)]
    beta_max = np.where(r <= d - 2, 0.5 * (v_up - v_dn), v_up)
    inside = (r >= d) | (f_dot <= r + PARITY_TOL) | (beta_max <= 0.0)
    cap = np.where(inside, 0.0, beta_max)

    # Kinks of beta -> f . clip(v - beta f): each coordinate enters the open
    # band (0,1) at one kink and leaves it at another; plus the ends 0, cap.
    enter = np.where(f > 0, v - 1.0, -v)
    leave = np.where(f > 0, v, 1.0 - v)
    kinks = np.concatenate([np.zeros((m, 1)), enter, leave, cap[:, None]], axis=1)
    kinks = np.minimum(np.maximum(kinks, 0.0), cap[:, None])
    kinks.sort(axis=1)
    shifted = np.clip(v[:, None, :] - kinks[:, :, None] * f[:, None, :], 0.0, 1.0)
    line = np.einsum("ijk,ik->ij", shifted, f)

    below = line <= r[:, None]
    first = np.argmax(below, axis=1)
    no_cross = first == 0          # line(0) = f_dot > r whenever the row is projected
    first = np.maximum(first, 1)
    b_lo, b_hi = kinks[idx, first - 1], kinks[idx, first]
    g_lo, g_hi = line[idx, first - 1], line[idx, first]
    drop = g_lo - g_hi
    interp = b_lo + (g_lo - r) * (b_hi - b_lo) / np.where(drop > 0.0, drop, 1.0)
    beta = np.where(no_cross, cap, np.where(drop > 0.0, interp, b_hi))

    z = np.clip(v - beta[:, None] * f, 0.0, 1.0)
    z = np.where(inside[:, None], cube, z)
    out = np.empty_like(z)
    out[idx[:, None], perm] = z
    return out


def membership(u, tol: float = PARITY_TOL) -> bool:
    """Parity-polytope membership within ``tol`` (parity_polytope.py:69-91):
    unit-cube test; r = even floor of the clipped l1 norm snapped up by
    PARITY_TOL (:62-64); two-slice weight alpha = clip((2 + r - s)/2, 0, 1);
    no upper slice when r + 2 > d unless alpha = 1; then every descending
    prefix sum must stay below alpha min(q, r) + (1 - alpha) min(q, r + 2)."""
    u = np.asarray(u, dtype=float)
    if u.ndim != 1 or u.size == 0:
        raise ValueError("membership expects a non-empty 1-D vector")
    d = u.size
    if np.any(u < -tol) or np.any(u > 1.0 + tol):
        return False
    s = min(max(float(u.sum()), 0.0), float(d))
    r = 2 * math.floor((s + PARITY_TOL) / 2.0)
    alpha = min(max((2.0 + r - s) / 2.0, 0.0), 1.0)
    if r + 2 > d and alpha < 1.0 - tol:
        return False
    prefix = np.cumsum(-np.sort(-u))
    q = np.arange(1, d + 1)
    bound = alpha * np.minimum(q, r) + (1.0 - alpha) * np.minimum(q, r + 2)
    return bool(np.all(prefix <= bound + tol))


# ---------------------------------------------------------------------------
# ADMM updates (admm_decoder.py:108-149) and the decode loop (:152-182)
# ---------------------------------------------------------------------------
def x_step(z, lam, gamma, g: Graph, p: Params) -> np.ndarray:
    """Variable update (admm_decoder.py:108-124): clipped average of the
    dual-adjusted replicas against the LLR step; degree-0 variables take the
    sign of their cost."""
    acc = np.bincount(g.edge_var, weights=z - lam / p.mu, minlength=g.n_vars)
    x = np.clip((acc - gamma / p.mu) / np.maximum(g.var_deg, 1), 0.0, 1.0)
    free = g.var_deg == 0
    if free.any():
        x[free] = (gamma[free] < 0.0).astype(float)
    return x


def z_step(x, z, lam, g: Graph, p: Params):
    """Replica update (admm_decoder.py:127-141): over-relaxed mixture
    w = rho x_gather + (1-rho) z, projection of w + lam/mu per check."""
    w = p.rho * x[g.edge_var] + (1.0 - p.rho) * z
    v = w + lam / p.mu
    z_new = np.empty_like(v)
    for rows in g.blocks.values():
        z_new[rows.reshape(-1)] = project_rows(v[rows]).reshape(-1)
    return z_new, w


def lam_step(lam, w, z_new, p: Params) -> np.ndarray:
    """Dual update (admm_decoder.py:144-149)."""
    return lam + p.mu * (w - z_new)


def is_codeword(g: Graph, bits) -> bool:
    """Even parity on every check (codes.py:145-154)."""
    b = np.asarray(bits).astype(np.int64)[g.edge_var]
    par = np.zeros(g.n_checks, dtype=np.int64)
    np.add.at(par, g.edge_check, b)
    return not bool(np.any(par & 1))


@dataclass(frozen=True)
class Result:
    x: np.ndarray
    status: str
    iterations: int
    integral: bool
    hard_decision: np.ndarray
    ml_certificate: bool


def finalize(x, status, t, g: Graph) -> Result:
    """Hard decision, integrality and ML certificate (admm_decoder.py:92-105)."""
    hard = (x > 0.5).astype(np.uint8)
    integral = bool(np.all(np.minimum(np.abs(x), np.abs(1.0 - x)) <= INTEGRALITY_TOL))
    return Result(x, status, t, integral, hard, integral and is_codeword(g, hard))


def decode(gamma, g: Graph, p: Params = Params()) -> Result:
    """ADMM decode of one frame (admm_decoder.py:152-182).

    Stops after iteration t when both the replica-to-variable residual and
    the replica movement fall strictly below eps^2 * E; the returned x is
    the one computed at the start of that iteration.
    """
    gamma = np.asarray(gamma, dtype=float)
    if gamma.shape != (g.n_vars,):
        raise ValueError(f"expected a length-{g.n_vars} LLR vector")
    if not np.all(np.isfinite(gamma)):
        raise ValueError("LLR vector must be finite")
    z = np.zeros(g.n_edges)
    lam = np.zeros(g.n_edges)
    thr = p.epsilon ** 2 * g.n_edges
    status, t_done, x = STATUS_MAX_ITERS, 0, np.zeros(g.n_vars)
    for t in range(1, p.t_max + 1):
        x = x_step(z, lam, gamma, g, p)
        z_new, w = z_step(x, z, lam, g, p)
        gx = x[g.edge_var]
        primal = float(((gx - z_new) ** 2).sum())
        moved = float(((z_new - z) ** 2).sum())
        lam = lam_step(lam, w, z_new, p)
        z = z_new
        t_done = t
        if primal < thr and moved < thr:
            status = STATUS_CONVERGED
            break
    return finalize(x, status, t_done, g)


def decode_many(gammas, g: Graph, p: Params = Params()) -> list[Result]:
    return [decode(row, g, p) for row in np.asarray(gammas, dtype=float)]


def _decode_chunk(args):
    n_vars, checks, gammas, p = args
    g = Graph(n_vars, checks)
    out = decode_many(gammas, g, p)
    return [(r.iterations, r.status == STATUS_CONVERGED, r.hard_decision) for r in out]


def decode_parallel(gammas, g: Graph, p: Params, workers: int | None = None):
    """Frame-parallel CPU decode over a process pool -- the reference
    harness's worker fan-out (simulator.py:194-220).  Returns
    (iterations[B], converged[B], hard[B, N])."""
    from concurrent.futures import ProcessPoolExecutor

    gammas = np.asarray(gammas, dtype=float)
    workers = workers or os.cpu_count() or 1
    if workers <= 1 or len(gammas) < 2 * workers:
        recs = _decode_chunk((g.n_vars, g.checks, gammas, p))
    else:
        chunks = np.array_split(gammas, workers * 4)
        payload = [(g.n_vars, g.checks, c, p) for c in chunks if len(c)]
        recs = []
        with ProcessPoolExecutor(max_workers=workers) as pool:
            for part in pool.map(_decode_chunk, payload):
                recs.extend(part)
    iters = np.array([r[0] for r in recs], dtype=np.int64)
    conv = np.array([r[1] for r in recs], dtype=bool)
    hard = np.stack([r[2] for r in recs]) if recs else np.zeros((0, g.n_vars), np.uint8)
    return iters, conv, hard


# ---------------------------------------------------------------------------
# Frame synthesis recipe (simulator.py:169-173, channels.py:73-110)
# ---------------------------------------------------------------------------
def awgn_sigma2(snr_db: float, rate: float) -> float:
    return 1.0 / (2.0 * rate * 10.0 ** (snr_db / 10.0))


def trial_gamma_awgn(n_vars: int, snr_db: float, rate: float, seed: int, point: int, trial: int):
    """All-zero codeword over BPSK/AWGN, seeded like the reference harness."""
    rng = np.random.default_rng(np.random.SeedSequence(entropy=seed, spawn_key=(point, trial)))
    s2 = awgn_sigma2(snr_db, rate)
    y = np.ones(n_vars) + math.sqrt(s2) * rng.standard_normal(n_vars)
    return 2.0 * y / s2


def trial_gamma_bsc(n_vars: int, p: float, seed: int, point: int, trial: int):
    rng = np.random.default_rng(np.random.SeedSequence(entropy=seed, spawn_key=(point, trial)))
    flips = (rng.random(n_vars) < p).astype(float)
    return (1.0 - 2.0 * flips) * math.log((1.0 - p) / p)
