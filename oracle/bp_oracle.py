"""CPU oracle for the BP baseline -- TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference's flooding sum-product decoder
(``polylp.bp_decoder``, /root/reference/pkg/src/polylp/bp_decoder.py) used
as the checker of the GPU BP kernel (csrc/bp.cuh).  Nothing in the product
package imports it; only ``tests/`` may.

Pinning: ``tests/test_oracle.py`` compares it bit for bit with the outputs
of the reference itself stored in ``tests/golden/bp.npz`` (made by
``tests/golden/make_golden.py``).  The arithmetic follows the reference's
operation order: totals by an edge-order accumulation (np.bincount), the
leave-one-out products as a left running product times a right running
product (np.cumprod order), and numpy's tanh / arctanh.
"""

from __future__ import annotations

import numpy as np

from .admm_oracle import Graph

ATANH_GUARD = 1.0 - 1e-15  # bp_decoder.py:19


def _edge_sum(g: Graph, w: np.ndarray) -> np.ndarray:
    """Per-variable sum of edge weights in edge order (np.bincount semantics)."""
    return np.bincount(g.edge_var, weights=w, minlength=g.n_vars)


def check_update(v2c: np.ndarray, g: Graph, clip: float) -> np.ndarray:
    """tanh-rule check-to-variable messages (bp_decoder.py:37-52)."""
    th = np.tanh(np.clip(0.5 * v2c, -0.5 * clip, 0.5 * clip))
    out = np.empty_like(v2c)
    for rows in g.blocks.values():  # rows: (m_d, d) edge ids of the degree-d checks
        t = th[rows]
        m, d = t.shape
        left = np.ones((m, d))
        right = np.ones((m, d))
        for k in range(1, d):  # running products, one multiply per step
            left[:, k] = t[:, 0] if k == 1 else left[:, k - 1] * t[:, k - 1]
        for k in range(d - 2, -1, -1):
            right[:, k] = t[:, d - 1] if k == d - 2 else right[:, k + 1] * t[:, k + 1]
        prod = np.clip(left * right, -ATANH_GUARD, ATANH_GUARD)
        out[rows.reshape(-1)] = np.clip(2.0 * np.arctanh(prod), -clip, clip).reshape(-1)
    return out


def posterior_llrs(gamma, g: Graph, t_max: int = 1000, llr_clip: float = 30.0, early_stop: bool = True):
    """Flooding BP (bp_decoder.py:55-95): returns (beliefs, iterations, found)."""
    gamma = np.asarray(gamma, dtype=float)
    c2v = np.zeros(g.n_edges)
    beliefs = gamma.copy()
    iterations, found = 0, False
    for t in range(1, t_max + 1):
        iterations = t
        totals = gamma + _edge_sum(g, c2v)
        v2c = np.clip(totals[g.edge_var] - c2v, -llr_clip, llr_clip)
        c2v = check_update(v2c, g, llr_clip)
        beliefs = gamma + _edge_sum(g, c2v)
        if early_stop and np.all(beliefs != 0.0):
            hard = (beliefs < 0.0).astype(np.int64)
            par = np.zeros(g.n_checks, dtype=np.int64)
            np.add.at(par, g.edge_check, hard[g.edge_var])
            if not np.any(par & 1):
                found = True
                break
    return beliefs, iterations, found


def decode_bp(gamma, g: Graph, t_max: int = 1000, llr_clip: float = 30.0, early_stop: bool = True):
    """decode_bp (bp_decoder.py:98-112): (p_one, hard, integral, iterations, found)."""
    b, it, found = posterior_llrs(gamma, g, t_max, llr_clip, early_stop)
    p_one = 0.5 * (1.0 - np.tanh(0.5 * b))
    hard = (b < 0.0).astype(np.uint8)
    integral = bool(np.all(np.minimum(p_one, 1.0 - p_one) <= 1e-5))
    return p_one, hard, integral, it, found
