"""The cut-search formulation of the parity-polytope projection
(csrc/projection.cuh, project_pp_cut) restated in numpy and checked against
the oracle's project_rows (the reference's two-slice algorithm,
parity_polytope.py:352-421) on the CPU: pins the MATH the kernels rely on --
the candidate facet from the signs of u - 1/2 with the closest coordinate
moved, the water-filling prefixes from one sort of |u - 1/2|, no facet test
and no beta_max cap -- independently of any GPU.  The kernels themselves are
checked against the reference goldens in test_gpu_projection.py."""
import numpy as np
import pytest

from oracle import admm_oracle as O


def cut_project(u, dt=np.float64):
    """project_pp_cut step by step (generic variant; `dt` the arithmetic)."""
    u = np.asarray(u, dtype=dt)
    _, d = u.shape
    half = dt(0.5)
    dk = u - half
    below = np.signbit(dk)
    even = ((d - below.sum(1)) % 2) == 0            # |T| even: move the closest coordinate
    t = np.sort(np.abs(dk), axis=1)
    p = half + np.where(even, -t[:, 0], t[:, 0])     # P_1 = 1 + s_(1)
    beta = p.copy()
    for j in range(1, d):
        p = p + (t[:, j] - half)
        beta = np.minimum(beta, p * dt(1.0 / (j + 1)))
    beta = np.maximum(beta, dt(0))
    te = np.where(even, t[:, 0], dt(-1))
    up = (dk >= 0) != (np.abs(dk) == te[:, None])
    return np.clip(np.where(up, u - beta[:, None], u + beta[:, None]), 0, 1)


def rows_for(d, rng):
    vert = rng.integers(0, 2, size=(3000, d)).astype(float)
    return np.concatenate([
        rng.uniform(-2, 3, (4000, d)),
        rng.normal(0.5, 0.6, (4000, d)),
        vert + rng.normal(0, 0.2, size=(3000, d)),           # near the vertices (the decoder's regime)
        np.clip(rng.normal(0.5, 0.5, (2000, d)), 0, 1),      # inside the cube
        rng.integers(-1, 3, (500, d)).astype(float),         # exact ties
        np.round(rng.uniform(-1, 2, (500, d)) * 4) / 4,
    ])


@pytest.mark.parametrize("d", [1, 2, 3, 4, 5, 6, 7, 8, 13, 16, 32])
def test_cut_search_equals_two_slice_projection_f64(d):
    rows = rows_for(d, np.random.default_rng(d))
    assert np.abs(cut_project(rows) - O.project_rows(rows)).max() <= 2e-15


@pytest.mark.parametrize("d", [3, 6, 13])
def test_cut_search_f32_arithmetic_is_at_rounding_level(d):
    rows = rows_for(d, np.random.default_rng(50 + d)).astype(np.float32)
    got = cut_project(rows, np.float32).astype(float)
    assert np.abs(got - O.project_rows(rows.astype(float))).max() <= 1e-6


def test_padded_rows_project_like_the_short_row():
    """-inf padding (the generic kernels' degree buckets): |d| = inf sorts last,
    never enters a prefix minimum, and the padded slots come out 0."""
    rng = np.random.default_rng(7)
    for d, bucket in ((3, 4), (5, 6), (9, 13)):
        rows = rng.normal(0.5, 0.7, (2000, d))
        padded = np.full((2000, bucket), -np.inf)
        padded[:, :d] = rows
        with np.errstate(invalid="ignore"):
            got = cut_project(padded)
        assert np.all(got[:, d:] == 0)
        assert np.abs(got[:, :d] - O.project_rows(rows)).max() <= 2e-15
