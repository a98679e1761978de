"""Drop-in conformance on the GPU: the reference's own decode properties and
acceptance criteria run against this package's decoder, step API and
membership kernel ("drop-in conformance").

Expected values that need the reference's scipy/brute-force test oracles
(LP optimum, codebook, ML words) or the reference itself were recorded in
the build container by tests/golden/make_golden.py (`conformance`,
`membership`); /root/reference does not exist on the GPU box.
"""
import numpy as np
import pytest
import torch

from conftest import load_golden

pytestmark = pytest.mark.gpu


def _code(f, name):
    from paper_1204_0556_b200 import ParityCheckMatrix

    ptr, ev = f[f"{name}_check_ptr"], f[f"{name}_edge_var"]
    return ParityCheckMatrix(int(f[f"{name}_n_vars"]), [ev[ptr[j]:ptr[j + 1]] for j in range(len(ptr) - 1)])


@pytest.fixture(scope="module")
def conf():
    return load_golden("conformance.npz")


# ---------------------------------------------------------------------------
# A12: membership (parity_polytope.py:69-91)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("d", range(1, 11))
def test_membership_kernel_matches_reference(cuda_ok, d):
    from paper_1204_0556_b200 import membership, membership_batch

    f = load_golden("membership.npz")
    rows = f[f"in_d{d}"]
    assert np.array_equal(membership_batch(rows), f[f"out_d{d}"])
    assert np.array_equal(membership_batch(rows, 1e-7), f[f"out7_d{d}"])
    k = int(np.argmax(f[f"out_d{d}"]))
    assert membership(rows[k]) is True
    with pytest.raises(ValueError):
        membership(np.zeros(0))


def test_projection_lands_in_polytope(cuda_ok):
    """Every projected row is a member (test_acceptance.py:83-117: membership(z, 1e-7))."""
    from paper_1204_0556_b200 import membership_batch, project_batch

    rng = np.random.default_rng(102)
    for d in range(1, 14):
        z = project_batch(rng.uniform(-2.0, 3.0, (2000, d)))
        assert membership_batch(z, 1e-7).all()


# ---------------------------------------------------------------------------
# Step API (admm_decoder.py:47-149)
# ---------------------------------------------------------------------------
def test_step_api_matches_reference_state_dumps(cuda_ok):
    """x, z, lambda after 1-3 hand-driven iterations (steps.npz, the
    reference's AdmmState); x- and lambda-updates are exact expressions."""
    from conftest import golden_code
    from paper_1204_0556_b200 import AdmmConfig, AdmmState, lambda_update, x_update, z_update

    f = load_golden("steps.npz")
    code = golden_code(f)
    st = AdmmState.initial(code)
    cfg = AdmmConfig(mu=5.0)
    for t in (1, 2, 3):
        x_update(st, code, f["gamma"], cfg)
        z_update(st, code, cfg)
        lambda_update(st, code, cfg)
        assert isinstance(st.x, np.ndarray) and st.x.dtype == np.float64
        assert np.abs(st.x - f[f"x{t}"]).max() <= 1e-12
        assert np.abs(st.z - f[f"z{t}"]).max() <= 1e-12
        assert np.abs(st.lam - f[f"lam{t}"]).max() <= 1e-12
    st0 = AdmmState.initial(code)
    x_update(st0, code, f["gamma"], cfg)
    assert np.array_equal(st0.x, f["x1"])  # bit-identical first x-update


def test_step_api_batched_device_state_matches_fused_decoder(cuda_ok):
    """The step kernels on a [B, E] CUDA state reproduce the fused decoder's
    fixed-iteration x (both fp64), and run at n = 16384 where the streaming
    engines keep no reference-order state."""
    from paper_1204_0556_b200 import (AdmmConfig, AdmmState, baseline_code, decode_batch, lambda_update,
                                      trial_gammas, x_update, z_update, Awgn, run_iterations)

    for key, T in (("cfg1_n96", 40), ("cfg5_n16384", 12)):
        code = baseline_code(key)
        gam = trial_gammas(code.n_vars, Awgn(2.5, code.design_rate), 1, 0, range(6))
        cfg = AdmmConfig(mu=5.0, epsilon=1e-300, t_max=T)
        st = AdmmState.initial(code, batch=6, device="cuda")
        g = torch.as_tensor(gam, device="cuda")
        for _ in range(T):
            x_update(st, code, g, cfg)
            z_update(st, code, cfg)
            lambda_update(st, code, cfg)
        assert st.x.shape == (6, code.n_vars) and st.x.is_cuda
        res = decode_batch(gam, code, cfg, dtype=torch.float64)
        assert np.abs(st.x.cpu().numpy() - res.x.cpu().numpy()).max() <= 1e-9
        x1, z1, l1 = run_iterations(gam[0], code, cfg, T)
        assert np.abs(x1 - st.x[0].cpu().numpy()).max() <= 1e-9
        assert np.abs(z1 - st.z[0].cpu().numpy()).max() <= 1e-9


def test_feasibility_at_convergence(cuda_ok, conf):
    """test_admm.py:147-168 with this package's AdmmState and step kernels:
    the loop converges, every check's replica lies in PP_d (membership
    kernel, tol 1e-5) and agrees with the gathered x; the final replicas
    match the reference's."""
    from paper_1204_0556_b200 import AdmmConfig, AdmmState, lambda_update, membership, x_update, z_update

    code = _code(conf, "c48")
    gamma = conf["feas_gamma"]
    cfg = AdmmConfig()
    st = AdmmState.initial(code)
    thr = cfg.epsilon ** 2 * code.n_edges
    for t in range(cfg.t_max):
        x_update(st, code, gamma, cfg)
        z_update(st, code, cfg)
        gathered = st.x[code.edge_var]
        primal = float(((gathered - st.z) ** 2).sum())
        moved = float(((st.z - st.z_prev) ** 2).sum())
        lambda_update(st, code, cfg)
        if primal < thr and moved < thr:
            break
    assert primal < thr
    assert t + 1 == int(conf["feas_iterations"])
    for j in range(code.n_checks):
        sl = code.check_slice(j)
        d = sl.stop - sl.start
        assert membership(st.z[sl], 1e-5)
        assert np.abs(gathered[sl] - st.z[sl]).max() <= 10 * cfg.epsilon * np.sqrt(d)
    assert np.abs(st.z - conf["feas_z"]).max() <= 1e-9
    assert np.abs(st.x - conf["feas_x"]).max() <= 1e-9


# ---------------------------------------------------------------------------
# Decode properties (test_admm.py:116-206)
# ---------------------------------------------------------------------------
def test_hamming_one_flip_matches_lp_and_ml(cuda_ok, conf):
    """test_admm.py:116-135: every <= 1-flip pattern reaches the LP optimum;
    flips on variables of degree >= 2 decode to the ML word with a
    certificate."""
    from paper_1204_0556_b200 import ParityCheckMatrix, decode

    lens, flat = conf["ham_check_len"], conf["ham_checks"]
    rows, k = [], 0
    for n in lens:
        rows.append(flat[k:k + n])
        k += n
    code = ParityCheckMatrix(7, rows)
    flips = [None, 0, 1, 2, 3, 4, 5, 6]
    for i, flip in enumerate(flips):
        gamma = conf["ham_gamma"][i]
        out = decode(gamma, code)
        assert float(gamma @ out.x) == pytest.approx(float(conf["ham_lp"][i]), abs=1e-3)
        assert np.abs(out.x - conf["ham_x"][i]).max() <= 1e-9
        if flip is None or conf["ham_var_deg"][flip] >= 2:
            assert out.integral
            assert np.array_equal(out.hard_decision, conf["ham_ml"][i])
            assert out.ml_certificate


def test_ml_certificate_against_codebook(cuda_ok, conf):
    """test_admm.py:170-184: every certified output is an ML codeword
    (cost against the whole codebook), on a batch decode; iteration counts
    and certificates equal the reference's."""
    from paper_1204_0556_b200 import decode_batch

    code = _code(conf, "c16")
    gam = conf["c16_gamma"]
    res = decode_batch(gam, code, dtype=torch.float64, want_hard=True)
    hard = res.hard.cpu().numpy().astype(float)
    cert = res.ml_certificate.cpu().numpy()
    assert np.array_equal(cert, conf["c16_cert"])
    assert np.array_equal(res.iterations.cpu().numpy(), conf["c16_iterations"])
    cost = (gam * hard).sum(1)
    assert np.all(cost[cert] <= conf["c16_best"][cert] + 1e-6)
    assert cert.sum() > 100


def test_objective_approaches_lp_value(cuda_ok, conf):
    """test_admm.py:186-197: gamma . x approaches the LP value (gap <= 1e-3
    at 1000 iterations, non-increasing from 100)."""
    from paper_1204_0556_b200 import AdmmConfig, decode

    code = _code(conf, "c24")
    gamma, lp = conf["lp24_gamma"], float(conf["lp24_value"])
    gaps = []
    for t, key in ((100, "lp24_x100"), (1000, "lp24_x1000")):
        out = decode(gamma, code, AdmmConfig(epsilon=1e-14, t_max=t, rho=1.0))
        assert np.abs(out.x - conf[key]).max() <= 1e-9
        gaps.append(abs(float(gamma @ out.x) - lp))
    assert gaps[1] <= gaps[0] + 1e-9
    assert gaps[1] <= 1e-3


def test_scaling_equivariance(cuda_ok):
    """test_admm.py:199-206: (gamma, mu) and (s gamma, s mu) give the same x."""
    from paper_1204_0556_b200 import AdmmConfig, decode, gen_regular_ldpc

    code = gen_regular_ldpc(24, 3, 6, seed=6)
    gamma = np.random.default_rng(7).normal(0.3, 1.0, 24)
    s = 3.7
    base = decode(gamma, code, AdmmConfig(mu=3.0, t_max=50, epsilon=1e-14))
    scaled = decode(s * gamma, code, AdmmConfig(mu=3.0 * s, t_max=50, epsilon=1e-14))
    assert np.abs(base.x - scaled.x).max() <= 1e-9


def test_determinism_and_batch_invariance(cuda_ok):
    """test_admm.py:139-145 (determinism), and a frame's result does not
    depend on the batch it is decoded in."""
    from paper_1204_0556_b200 import decode, decode_batch, gen_regular_ldpc

    code = gen_regular_ldpc(48, 3, 6, seed=4)
    rng = np.random.default_rng(0)
    gamma = rng.normal(0.5, 1.0, (37, 48))
    a, b = decode(gamma[3], code), decode(gamma[3], code)
    assert np.array_equal(a.x, b.x) and a.iterations == b.iterations
    res = decode_batch(gamma, code)
    assert np.array_equal(res.x[3].cpu().numpy(), a.x)


# ---------------------------------------------------------------------------
# Acceptance criteria 5-7 (test_acceptance.py:186-262) on the GPU decoder
# ---------------------------------------------------------------------------
def _crit_gammas(code, p, seed, n):
    from paper_1204_0556_b200 import Bsc, trial_gammas

    return trial_gammas(code.n_vars, Bsc(p), seed, 0, range(n))


def test_criterion_05_convergence_behavior(cuda_ok, conf):
    from paper_1204_0556_b200 import AdmmConfig, decode_batch

    code = _code(conf, "c96")
    gam = _crit_gammas(code, 0.02, 105, 2000)
    res = decode_batch(gam, code, AdmmConfig(), dtype=torch.float64)
    it = res.iterations.cpu().numpy()
    w = res.weight.cpu().numpy()
    assert np.array_equal(it, conf["crit5_iterations"])
    assert np.array_equal(w, conf["crit5_weight"])
    correct = it[w == 0]
    assert (correct < 200).mean() >= 0.95
    assert correct.mean() <= AdmmConfig().t_max / 5


def test_criterion_06_over_relaxation_speedup(cuda_ok, conf):
    from paper_1204_0556_b200 import AdmmConfig, decode_batch

    code = _code(conf, "c96")
    gam = _crit_gammas(code, 0.02, 106, 1000)
    it = {}
    for rho, key in ((1.0, "crit6_iter_rho1"), (1.9, "crit6_iter_rho19")):
        it[rho] = decode_batch(gam, code, AdmmConfig(rho=rho), dtype=torch.float64).iterations.cpu().numpy()
        assert np.array_equal(it[rho], conf[key])
    assert it[1.9].sum() / it[1.0].sum() <= 0.8


def test_criterion_07_parameter_robustness(cuda_ok, conf):
    """WER agreement within 2 s.e. across mu and epsilon, through the GPU
    harness (run_point); word and bit errors equal the reference's."""
    from paper_1204_0556_b200 import AdmmConfig, Bsc, DecoderRef, run_point

    code = _code(conf, "c96")
    wer = {}
    for tag, cfg, pt in (("mu3", AdmmConfig(mu=3.0), 0), ("mu7", AdmmConfig(mu=7.0), 0),
                         ("eps4", AdmmConfig(epsilon=1e-4), 1), ("eps6", AdmmConfig(epsilon=1e-6), 1)):
        s = run_point(code, Bsc(0.03), DecoderRef("admm", cfg), n_trials=5000, seed=107, point_index=pt)
        assert s.trials == int(conf[f"crit7_{tag}_trials"])
        assert s.word_errors == int(conf[f"crit7_{tag}_word_errors"])
        assert s.bit_errors == int(conf[f"crit7_{tag}_bit_errors"])
        wer[tag] = (s.wer, s.trials)

    def agree(a, b):
        (w1, n1), (w2, n2) = a, b
        return abs(w1 - w2) <= 2.0 * np.sqrt(w1 * (1 - w1) / n1 + w2 * (1 - w2) / n2)

    assert agree(wer["mu3"], wer["mu7"]) and agree(wer["eps4"], wer["eps6"])
