"""Pin the CPU oracle to the reference: golden vectors produced by the
reference package itself (tests/golden/make_golden.py) and the reference's
own known-answer tests.  CPU only."""
import numpy as np
import pytest

from conftest import golden_code, load_golden
from oracle import admm_oracle as O


def graph_of(f):
    return O.Graph.of(golden_code(f))


@pytest.mark.parametrize("d", range(1, 14))
def test_projection_matches_reference_golden(d):
    P = load_golden("projection.npz")
    got = O.project_rows(P[f"in_d{d}"])
    assert np.array_equal(got, P[f"out_d{d}"])  # bit-exact restatement


@pytest.mark.parametrize(
    "u,want",
    [  # test_parity_polytope.py:139-157
        ([1, 1, 0, 0], [1, 1, 0, 0]),
        ([1, 0, 0], [2 / 3, 1 / 3, 1 / 3]),
        ([1, -0.2], [0.4, 0.4]),
        ([0, 0, 1], [1 / 3, 1 / 3, 2 / 3]),
        ([0.7], [0.0]),
        ([-3.0], [0.0]),
    ],
)
def test_projection_kats(u, want):
    assert np.allclose(O.project_rows(np.array([u], float))[0], want, atol=1e-9)


def test_projection_domain_errors():
    with pytest.raises(ValueError):
        O.project_rows(np.array([[np.nan, 0.0]]))
    with pytest.raises(ValueError):
        O.project_rows(np.zeros((3, 0)))


def _decode_frames(f, n):
    g = graph_of(f)
    rate = 1.0 - g.n_checks / g.n_vars
    gam = np.array([O.trial_gamma_awgn(g.n_vars, float(f["snr_db"]), rate, 1, 0, t) for t in range(n)])
    p = O.Params(mu=float(f["mu"]), epsilon=float(f["epsilon"]), t_max=int(f["t_max"]), rho=float(f["rho"]))
    return g, gam, O.decode_many(gam, g, p)


@pytest.mark.parametrize("name,n", [("decode_cfg1.npz", 120), ("decode_cfg2.npz", 6), ("decode_cfg4.npz", 12)])
def test_decode_matches_reference_golden(name, n):
    f = load_golden(name)
    g, gam, res = _decode_frames(f, n)
    k = min(n, len(f["gamma_head"]))
    assert np.array_equal(gam[:k], f["gamma_head"][:k])  # frame synthesis is bit-identical
    hard = np.unpackbits(f["hard"], axis=1)[:n, : g.n_vars]
    for t, r in enumerate(res):
        assert r.iterations == f["iterations"][t]
        assert r.status == (O.STATUS_CONVERGED if f["converged"][t] else O.STATUS_MAX_ITERS)
        assert r.integral == bool(f["integral"][t])
        assert r.ml_certificate == bool(f["certificate"][t])
        assert np.array_equal(r.hard_decision, hard[t])
        if t < len(f["x"]):
            assert np.array_equal(r.x, f["x"][t])


def test_fixed_iteration_state_matches_reference_golden():
    f = load_golden("fixed_cfg1.npz")
    g = graph_of(f)
    for T in (1, 50):
        p = O.Params(mu=5.0, epsilon=1e-300, t_max=T)
        for k in range(4):
            r = O.decode(f["gamma"][k], g, p)
            assert r.iterations == T
            assert np.array_equal(r.x, f[f"x_T{T}"][k])


def test_step_dumps_match_reference_golden():
    f = load_golden("steps.npz")
    g = graph_of(f)
    p = O.Params(mu=5.0)
    z = np.zeros(g.n_edges)
    lam = np.zeros(g.n_edges)
    for t in range(1, 4):
        x = O.x_step(z, lam, f["gamma"], g, p)
        z_new, w = O.z_step(x, z, lam, g, p)
        lam = O.lam_step(lam, w, z_new, p)
        z = z_new
        assert np.array_equal(x, f[f"x{t}"])
        assert np.array_equal(z, f[f"z{t}"])
        assert np.array_equal(lam, f[f"lam{t}"])


def test_update_step_kats():
    # test_admm.py:27-46: three checks on one pair of variables
    g = O.Graph(2, [[0, 1], [0, 1], [0, 1]])
    p = O.Params(mu=3.0)
    z = np.zeros(6)
    assert np.all(O.x_step(z, z, np.array([6.0, 6.0]), g, p) == 0.0)
    assert np.all(O.x_step(np.ones(6), z, np.array([-6.0, -6.0]), g, p) == 1.0)
    assert np.allclose(O.x_step(np.full(6, 0.5), z, np.zeros(2), g, p), 0.5)
    # test_admm.py:75-81: lambda arithmetic
    lam = O.lam_step(np.zeros(3), np.array([0.6, 0.4, 0.5]), np.array([0.5, 0.5, 0.5]), p)
    assert np.allclose(lam, [0.3, -0.3, 0.0], atol=1e-12)


def test_single_check_fixture():
    # test_admm.py:94-102
    g = O.Graph(4, [[0, 1, 2, 3]])
    r = O.decode(np.array([2.2, 2.2, -1.0, 2.2]), g, O.Params())
    assert r.status == O.STATUS_CONVERGED and r.integral and r.ml_certificate
    assert np.allclose(r.x, 0.0, atol=1e-4)


def test_params_validation():
    for kw in ({"mu": 0.0}, {"rho": 2.0}, {"epsilon": -1.0}, {"t_max": 0}):
        with pytest.raises(ValueError):
            O.Params(**kw)


@pytest.mark.parametrize("d", range(1, 11))
def test_membership_matches_reference_golden(d):
    """membership() restatement (parity_polytope.py:69-91) against the
    reference's answers on inside / outside / boundary rows, two tolerances."""
    f = load_golden("membership.npz")
    rows = f[f"in_d{d}"]
    assert np.array_equal([O.membership(u) for u in rows], f[f"out_d{d}"])
    assert np.array_equal([O.membership(u, 1e-7) for u in rows], f[f"out7_d{d}"])
    assert f[f"out_d{d}"].any() and not f[f"out_d{d}"].all()  # both outcomes exercised


def test_membership_rejects_empty():
    with pytest.raises(ValueError):
        O.membership(np.zeros(0))


@pytest.mark.parametrize("name", ["sweep_cfg2_3p0.npz", "sweep_cfg4_5p0.npz", "sweep_cfg5_bsc.npz"])
def test_oracle_reproduces_sweep_endpoint_golden(name):
    """The round-2 sweep fixtures (reference outputs) against the oracle on
    their first frames: same frame recipe, iterations, hard decisions, x."""
    f = load_golden(name)
    g = graph_of(f)
    n = g.n_vars
    p = O.Params(mu=float(f["mu"]), epsilon=float(f["epsilon"]), t_max=int(f["t_max"]), rho=float(f["rho"]))
    rate = 1.0 - g.n_checks / n
    want = np.unpackbits(f["hard"], axis=1)[:, :n]
    for t in range(2 if "cfg5" in name else 4):
        if str(f["channel"]) == "bsc":
            gam = O.trial_gamma_bsc(n, float(f["param"]), int(f["seed"]), int(f["point"]), t)
        else:
            gam = O.trial_gamma_awgn(n, float(f["param"]), rate, int(f["seed"]), int(f["point"]), t)
        r = O.decode(gam, g, p)
        assert r.iterations == f["iterations"][t]
        assert np.array_equal(r.hard_decision, want[t])
        assert np.array_equal(r.x, f["x"][t])
