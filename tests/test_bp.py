"""BP baseline: oracle pinned to the reference, GPU kernel
checked against both.  Mirrors the reference's tests/test_bp.py cases."""

import numpy as np
import pytest

from conftest import load_golden
from oracle import admm_oracle as O
from oracle import bp_oracle as B


def _graph(n, lens, flat):
    checks, pos = [], 0
    for d in lens:
        checks.append(flat[pos:pos + d])
        pos += d
    return O.Graph(int(n), checks)


def _code(n, lens, flat):
    from paper_1204_0556_b200 import ParityCheckMatrix

    g = _graph(n, lens, flat)
    return ParityCheckMatrix(g.n_vars, [c.tolist() for c in g.checks])


def _c1():
    f = load_golden("bp.npz")
    ptr, ev = f["c1_check_ptr"], f["c1_edge_var"]
    return f, _graph(int(f["c1_n_vars"]), np.diff(ptr), ev), np.diff(ptr), ev


# ---------------------------------------------------------------------------
# oracle vs the reference's own outputs (CPU)
# ---------------------------------------------------------------------------
def test_oracle_matches_reference_bp_bit_exactly():
    f, g, _, _ = _c1()
    for k in range(0, 200, 7):
        b, it, fd = B.posterior_llrs(f["c1_gamma"][k], g)
        assert np.array_equal(b, f["c1_beliefs"][k])
        assert it == f["c1_iterations"][k] and fd == f["c1_found"][k]
        x, _, integ, _, _ = B.decode_bp(f["c1_gamma"][k], g)
        assert np.array_equal(x, f["c1_x"][k]) and integ == f["c1_integral"][k]
    for T in (1, 5, 30):
        for k in range(16):
            b, _, _ = B.posterior_llrs(f["c1_gamma"][k], g, t_max=T, early_stop=False)
            assert np.array_equal(b, f[f"c1_fixed_T{T}"][k])


def test_oracle_mixed_degrees_and_trees():
    f = load_golden("bp.npz")
    g = _graph(40, f["mx_checks"], f["mx_flat"])
    for k in range(len(f["mx_gamma"])):
        b, _, _ = B.posterior_llrs(f["mx_gamma"][k], g, t_max=7, llr_clip=12.0, early_stop=False)
        assert np.array_equal(b, f["mx_beliefs_T7"][k])
        b, it, fd = B.posterior_llrs(f["mx_gamma"][k], g, t_max=60)
        assert np.array_equal(b, f["mx_beliefs"][k]) and it == f["mx_iterations"][k] and fd == f["mx_found"][k]
    for k in range(25):
        g = _graph(f[f"tree{k}_n"], f[f"tree{k}_lens"], f[f"tree{k}_flat"])
        b, _, _ = B.posterior_llrs(f[f"tree{k}_gamma"], g, t_max=40, llr_clip=500.0, early_stop=False)
        assert np.array_equal(b, f[f"tree{k}_beliefs"])
        assert np.abs(b - f[f"tree{k}_exact"]).max() <= 1e-6  # BP is exact on trees


def test_bp_config_validation_and_refs():
    from paper_1204_0556_b200 import BpConfig, DecoderRef

    with pytest.raises(ValueError):
        BpConfig(t_max=0)
    with pytest.raises(ValueError):
        BpConfig(llr_clip=0.0)
    assert DecoderRef("bp").admm_config() == BpConfig()


# ---------------------------------------------------------------------------
# GPU kernel
# ---------------------------------------------------------------------------
@pytest.mark.gpu
def test_gpu_bp_fixed_iterations_match_reference(cuda_ok):
    import torch

    from paper_1204_0556_b200 import BpConfig, decode_bp_batch

    f, _, lens, ev = _c1()
    code = _code(int(f["c1_n_vars"]), lens, ev)
    for T in (1, 5, 30):
        r = decode_bp_batch(f["c1_gamma"][:16], code, BpConfig(t_max=T, early_stop=False), dtype=torch.float64)
        got = r.beliefs.cpu().numpy()
        want = f[f"c1_fixed_T{T}"]
        # GPU tanh/atanh agree with libm to an ulp and the schedule is the
        # reference's, but atanh near the +-(1 - 1e-15) guard amplifies an ulp
        # of its argument by 1 / (1 - prod^2): beliefs agree to 1e-6 relative
        # (one iteration: 1e-12)
        tol = 1e-12 if T == 1 else 1e-6
        assert np.abs(got - want).max() <= tol * max(1.0, np.abs(want).max())
        assert (r.iterations.cpu().numpy() == T).all()


@pytest.mark.gpu
def test_gpu_bp_early_stop_matches_reference(cuda_ok):
    import torch

    from paper_1204_0556_b200 import BpConfig, decode_bp_batch

    f, _, lens, ev = _c1()
    code = _code(int(f["c1_n_vars"]), lens, ev)
    r = decode_bp_batch(f["c1_gamma"], code, BpConfig(), dtype=torch.float64)
    torch.cuda.synchronize()
    assert np.array_equal(r.iterations.cpu().numpy(), f["c1_iterations"])
    assert np.array_equal(r.found.cpu().numpy(), f["c1_found"].astype(bool))
    b = r.beliefs.cpu().numpy()
    fd = f["c1_found"].astype(bool)
    # frames that stopped on a codeword: same decision, beliefs to 1e-6
    assert np.array_equal(b[fd] < 0, f["c1_beliefs"][fd] < 0)
    assert np.abs(b[fd] - f["c1_beliefs"][fd]).max() <= 1e-6 * max(1.0, np.abs(f["c1_beliefs"][fd]).max())
    assert np.abs(r.x.cpu().numpy()[fd] - f["c1_x"][fd]).max() <= 1e-9
    assert np.array_equal(((r.flags & 2) != 0).cpu().numpy()[fd], f["c1_integral"].astype(bool)[fd])
    # frames that ran all 1000 iterations without a codeword: saturated BP
    # oscillates, and an ulp of tanh/atanh can move individual bits after
    # hundreds of iterations -- same iteration count and failure, and most
    # hard decisions equal
    assert (r.iterations.cpu().numpy()[~fd] == 1000).all()
    assert ((b[~fd] < 0) == (f["c1_beliefs"][~fd] < 0)).mean() >= 0.9


@pytest.mark.gpu
def test_gpu_bp_mixed_degrees_trees_and_cfg2(cuda_ok):
    import torch

    from paper_1204_0556_b200 import BpConfig, baseline_code, decode_bp_batch

    f = load_golden("bp.npz")
    code = _code(40, f["mx_checks"], f["mx_flat"])
    r = decode_bp_batch(f["mx_gamma"], code, BpConfig(t_max=7, early_stop=False, llr_clip=12.0))
    assert np.abs(r.beliefs.cpu().numpy() - f["mx_beliefs_T7"]).max() <= 1e-6 * 12
    r = decode_bp_batch(f["mx_gamma"], code, BpConfig(t_max=60))
    assert np.array_equal(r.iterations.cpu().numpy(), f["mx_iterations"])
    assert np.array_equal(r.found.cpu().numpy(), f["mx_found"].astype(bool))
    for k in range(25):
        tc = _code(f[f"tree{k}_n"], f[f"tree{k}_lens"], f[f"tree{k}_flat"])
        r = decode_bp_batch(f[f"tree{k}_gamma"], tc, BpConfig(t_max=40, llr_clip=500.0, early_stop=False))
        b = r.beliefs[0].cpu().numpy()
        assert np.abs(b - f[f"tree{k}_exact"]).max() <= 1e-6
        assert np.abs(b - f[f"tree{k}_beliefs"]).max() <= 1e-6 * max(1.0, np.abs(b).max())
    c2 = baseline_code("cfg2_n1008")
    r = decode_bp_batch(f["c2_gamma"], c2, BpConfig(t_max=200), dtype=torch.float64)
    assert np.array_equal(r.iterations.cpu().numpy(), f["c2_iterations"])
    assert np.array_equal(r.found.cpu().numpy(), f["c2_found"].astype(bool))
    hard = np.unpackbits(f["c2_hard"], axis=1)[:, :c2.n_vars]
    assert np.array_equal(r.hard.cpu().numpy(), hard)
    # fp32 throughput mode: same hard decisions on (nearly) every frame
    r32 = decode_bp_batch(f["c2_gamma"], c2, BpConfig(t_max=200), dtype=torch.float32)
    same = (r32.hard.cpu().numpy() == hard).all(axis=1).mean()
    assert same >= 0.95


@pytest.mark.gpu
def test_gpu_bp_reference_test_cases(cuda_ok):
    """The reference's tests/test_bp.py cases against the GPU kernel."""
    from paper_1204_0556_b200 import (STATUS_CONVERGED, STATUS_MAX_ITERS, BpConfig, ParityCheckMatrix,
                                      decode_bp, is_codeword, posterior_llrs)

    code = ParityCheckMatrix.from_dense([[1, 1, 0], [0, 1, 1]])
    out = decode_bp(np.zeros(3), code, BpConfig(t_max=9))
    assert out.status == STATUS_MAX_ITERS and out.iterations == 9 and not out.hard_decision.any()
    b, _, _ = posterior_llrs(np.zeros(3), code, BpConfig(t_max=9))
    assert np.all(b == 0.0)
    single = ParityCheckMatrix.from_dense([[1, 1, 1]])
    gamma = np.array([2.0, 2.0, -0.5])
    b, _, _ = posterior_llrs(gamma, single, BpConfig(t_max=1, early_stop=False))
    g = O.Graph(3, [[0, 1, 2]])
    assert np.abs(b - B.posterior_llrs(gamma, g, t_max=1, early_stop=False)[0]).max() <= 1e-12
    # odd symmetry of the check rule
    gamma = np.array([1.3, 0.8, 0.5])
    bp_, _, _ = posterior_llrs(gamma, single, BpConfig(t_max=1, early_stop=False))
    fl = gamma * np.array([1.0, 1.0, -1.0])
    bn, _, _ = posterior_llrs(fl, single, BpConfig(t_max=1, early_stop=False))
    ep, en = bp_ - gamma, bn - fl
    assert ep[2] == pytest.approx(en[2], abs=1e-12)
    assert ep[0] == pytest.approx(-en[0], abs=1e-12) and ep[1] == pytest.approx(-en[1], abs=1e-12)
    # saturation
    b, _, _ = posterior_llrs(np.array([200.0, 200.0]), ParityCheckMatrix.from_dense([[1, 1]]),
                             BpConfig(t_max=5, llr_clip=30.0))
    assert np.all(b <= 230.0)
    # soft output convention and early exit on a codeword
    out = decode_bp(np.array([4.0, 4.0, -6.0]), single, BpConfig(t_max=3))
    assert out.x[0] < 0.5 and (out.hard_decision == (out.x > 0.5)).all()
    rng = np.random.default_rng(1)
    for _ in range(20):
        out = decode_bp(rng.normal(0.5, 1.5, 3), single, BpConfig(t_max=50))
        if out.status == STATUS_CONVERGED:
            assert is_codeword(single, out.hard_decision)
    with pytest.raises(ValueError):
        decode_bp(np.ones(2), single)
    with pytest.raises(ValueError):
        decode_bp(np.array([1.0, np.nan, 0.0]), single)


@pytest.mark.gpu
def test_gpu_bp_harness_reproduces_reference_csv(cuda_ok):
    """DecoderRef('bp') through the batched GPU harness: the reference's CSV."""
    from paper_1204_0556_b200 import Awgn, BpConfig, Bsc, DecoderRef, stats_to_csv, sweep

    f, _, lens, ev = _c1()
    code = _code(int(f["c1_n_vars"]), lens, ev)
    got = stats_to_csv(sweep(code, [Bsc(0.04), Awgn(2.0, code.design_rate)], DecoderRef("bp", BpConfig(t_max=100)),
                             n_trials=200, seed=109, batch_size=64), timing=False)
    assert got == str(f["c1_csv_bp"])


@pytest.mark.gpu
def test_gpu_bp_batch_invariance(cuda_ok):
    import torch

    from paper_1204_0556_b200 import Awgn, BpConfig, baseline_code, decode_bp_batch, synth_llr

    code = baseline_code("cfg2_n1008")
    g = synth_llr(code.n_vars, Awgn(1.75, 0.5), seed=3, point=0, trial0=0, batch=700, dtype=torch.float32)
    a = decode_bp_batch(g, code, BpConfig(t_max=50), dtype=torch.float32)
    b = decode_bp_batch(g[350:], code, BpConfig(t_max=50), dtype=torch.float32)
    assert torch.equal(a.beliefs[350:], b.beliefs) and torch.equal(a.iterations[350:], b.iterations)
    assert torch.equal(a.hard, (a.beliefs < 0).to(torch.uint8))
