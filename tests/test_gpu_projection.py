"""K1 projection parity: the CUDA projection against the reference's
project_batch outputs (golden) and the oracle restatement."""
import numpy as np
import pytest
import torch

from conftest import load_golden
from oracle import admm_oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("d", range(1, 14))
def test_project_batch_f64_matches_reference_golden(cuda_ok, d):
    from paper_1204_0556_b200 import project_batch

    P = load_golden("projection.npz")
    got = project_batch(P[f"in_d{d}"])
    assert np.abs(got - P[f"out_d{d}"]).max() <= 1e-12


@pytest.mark.parametrize("d", [1, 2, 3, 5, 6, 7, 8, 9, 13, 14, 16, 17, 24, 32])
def test_project_batch_f64_matches_oracle_adversarial(cuda_ok, d):
    from paper_1204_0556_b200 import project_batch

    rng = np.random.default_rng(d)
    rows = np.concatenate([
        rng.uniform(-2, 3, (2000, d)),
        rng.integers(-1, 3, (500, d)).astype(float),
        np.round(rng.uniform(-1, 2, (500, d)) * 4) / 4,
        rng.normal(0.5, 0.6, (2000, d)),
    ])
    assert np.abs(project_batch(rows) - O.project_rows(rows)).max() <= 1e-12


@pytest.mark.parametrize("d", [3, 6, 13])
def test_project_batch_f32_close_to_oracle(cuda_ok, d):
    from paper_1204_0556_b200.parity_polytope import project_rows_device

    rng = np.random.default_rng(100 + d)
    rows = rng.uniform(-2, 3, (5000, d))
    got = project_rows_device(torch.tensor(rows, dtype=torch.float32, device="cuda")).double().cpu().numpy()
    want = O.project_rows(rows.astype(np.float32).astype(float))
    # fp32 rounding (~1e-7) plus the fp32 facet tolerance 1e-6 (csrc/common.cuh)
    assert np.abs(got - want).max() <= 5e-6


def test_project_batch_kats_and_errors(cuda_ok):
    from paper_1204_0556_b200 import project_batch

    for u, want in [([1, 1, 0, 0], [1, 1, 0, 0]), ([1, 0, 0], [2 / 3, 1 / 3, 1 / 3]),
                    ([1, -0.2], [0.4, 0.4]), ([0, 0, 1], [1 / 3, 1 / 3, 2 / 3]), ([0.7], [0.0])]:
        assert np.allclose(project_batch(np.array([u], float))[0], want, atol=1e-12)
    with pytest.raises(ValueError):
        project_batch(np.array([[np.nan, 0.0]]))
    with pytest.raises(ValueError):
        project_batch(np.zeros((2, 0)))
    assert project_batch(np.zeros((0, 3))).shape == (0, 3)


def test_projection_properties(cuda_ok):
    """Idempotence and permutation equivariance (test_acceptance.py:83-117)."""
    from paper_1204_0556_b200 import project_batch

    rng = np.random.default_rng(7)
    for d in (4, 6, 9):
        u = rng.uniform(-2, 3, (3000, d))
        z = project_batch(u)
        assert np.abs(project_batch(z) - z).max() <= 1e-9
        perm = rng.permutation(d)
        assert np.abs(project_batch(u[:, perm]) - z[:, perm]).max() <= 1e-12
