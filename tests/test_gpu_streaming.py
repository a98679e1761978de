"""Streaming engine (csrc/streaming.cuh) parity: forced onto the golden
codes, and automatically on codes too large for the resident engine
(BASELINE config 5, n = 16384), against the reference goldens / the oracle."""
import numpy as np
import pytest
import torch

from conftest import golden_code, load_golden
from oracle import admm_oracle as O

pytestmark = pytest.mark.gpu


def _frames(f, code, n, point=0):
    rate = 1.0 - code.n_checks / code.n_vars
    return np.array([O.trial_gamma_awgn(code.n_vars, float(f["snr_db"]), rate, 1, point, t) for t in range(n)])


@pytest.mark.parametrize("engine,kind", [("streaming", 3), ("wide", 3)])
@pytest.mark.parametrize("name", ["decode_cfg1.npz", "decode_cfg2.npz", "decode_cfg4.npz"])
def test_streaming_f64_matches_reference_golden(cuda_ok, name, engine, kind):
    from paper_1204_0556_b200 import AdmmConfig, decode_batch

    f = load_golden(name)
    code = golden_code(f)
    B = len(f["iterations"])
    gam = _frames(f, code, B)
    cfg = AdmmConfig(mu=float(f["mu"]), epsilon=float(f["epsilon"]), t_max=int(f["t_max"]), rho=float(f["rho"]))
    res = decode_batch(gam, code, cfg, dtype=torch.float64, want_hard=True, engine=engine)
    assert res.info["engine"] == kind
    assert (res.info["kernel"] == 5) == (engine == "wide")
    want_hard = np.unpackbits(f["hard"], axis=1)[:, : code.n_vars]
    fl = res.flags.cpu().numpy()
    assert np.array_equal(res.iterations.cpu().numpy(), f["iterations"])
    assert np.array_equal((fl & 1) != 0, f["converged"] != 0)
    assert np.array_equal((fl & 2) != 0, f["integral"] != 0)
    assert np.array_equal(((fl & 2) != 0) & ((fl & 4) != 0), f["certificate"] != 0)
    assert np.array_equal(res.hard.cpu().numpy(), want_hard)
    assert np.array_equal(res.weight.cpu().numpy(), want_hard.sum(1))
    nx = len(f["x"])
    assert np.abs(res.x[:nx].cpu().numpy() - f["x"]).max() <= 1e-9


@pytest.mark.parametrize("engine", ["streaming", "wide"])
def test_streaming_equals_resident_f32(cuda_ok, engine):
    from paper_1204_0556_b200 import AdmmConfig, baseline_code, decode_batch

    code = baseline_code("cfg2_n1008")
    g = torch.randn(200, code.n_vars, device="cuda", generator=torch.Generator("cuda").manual_seed(1)) * 2.5 + 3.2
    cfg = AdmmConfig(mu=5.0)
    a = decode_batch(g, code, cfg, dtype=torch.float32, engine="resident")
    b = decode_batch(g, code, cfg, dtype=torch.float32, engine=engine)
    same = (a.x > 0.5).eq(b.x > 0.5).all(dim=1).float().mean().item()
    assert same >= 0.995
    assert (a.iterations - b.iterations).abs().float().mean().item() <= 2.0


@pytest.mark.parametrize("engine", ["streaming", "wide"])
def test_streaming_irregular_and_zero_degree(cuda_ok, engine):
    from paper_1204_0556_b200 import AdmmConfig, ParityCheckMatrix, decode_batch

    codes = [
        ParityCheckMatrix.from_dense([[1, 1, 0, 1, 1, 0, 0], [1, 0, 1, 1, 0, 1, 0], [0, 1, 1, 1, 0, 0, 1]]),
        ParityCheckMatrix(6, [[0, 1, 2], [1, 2, 3, 4]]),
        ParityCheckMatrix(12, [list(range(0, 8)), list(range(4, 11)), [0, 7, 10]]),  # var 11: degree 0
    ]
    if engine == "streaming":
        codes.append(ParityCheckMatrix(20, [list(range(0, 9)), list(range(5, 20)), [0, 7, 19]]))
    rng = np.random.default_rng(4)
    for code in codes:
        gam = rng.normal(0.5, 1.2, (33, code.n_vars))
        res = decode_batch(gam, code, AdmmConfig(mu=3.0, t_max=300), dtype=torch.float64, engine=engine)
        g = O.Graph.of(code)
        for t in range(len(gam)):
            r = O.decode(gam[t], g, O.Params(mu=3.0, t_max=300))
            assert int(res.iterations[t]) == r.iterations
            assert np.abs(res.x[t].cpu().numpy() - r.x).max() <= 1e-9


@pytest.mark.parametrize("engine", ["auto", "streaming", "wide"])
def test_config5_large_block_matches_oracle(cuda_ok, engine):
    """n = 16384 does not fit one SM: the automatic engine is the cluster
    engine (fp64: 8-CTA clusters); the sharded and the wide kernels are
    forced too."""
    from paper_1204_0556_b200 import AdmmConfig, baseline_code, decode_batch

    code = baseline_code("cfg5_n16384")
    gam = np.stack([O.trial_gamma_bsc(code.n_vars, 0.04, 1, 0, t) for t in range(3)]
                   + [O.trial_gamma_awgn(code.n_vars, 2.5, 0.5, 1, 1, t) for t in range(3)])
    cfg = AdmmConfig(mu=5.0)
    res = decode_batch(gam, code, cfg, dtype=torch.float64, want_hard=True, engine=engine)
    assert res.info["engine"] == 3
    g = O.Graph.of(code)
    for t in range(len(gam)):
        r = O.decode(gam[t], g, O.Params(mu=5.0))
        assert int(res.iterations[t]) == r.iterations
        assert np.abs(res.x[t].cpu().numpy() - r.x).max() <= 1e-9
        assert np.array_equal(res.hard[t].cpu().numpy(), r.hard_decision)
    r32 = decode_batch(gam, code, cfg, dtype=torch.float32, want_hard=True, engine=engine)
    assert torch.equal(r32.hard, res.hard)
    # fixed iteration count (north star: fp64 x within 1e-9 after T iterations)
    fixed = AdmmConfig(mu=5.0, epsilon=1e-300, t_max=12)
    rt = decode_batch(gam[:2], code, fixed, dtype=torch.float64, engine=engine)
    for t in range(2):
        r = O.decode(gam[t], g, O.Params(mu=5.0, epsilon=1e-300, t_max=12))
        assert int(rt.iterations[t]) == 12 == r.iterations
        assert np.abs(rt.x[t].cpu().numpy() - r.x).max() <= 1e-9


@pytest.mark.parametrize("engine", ["streaming", "wide"])
def test_streaming_rejects_state_io(cuda_ok, engine):
    from paper_1204_0556_b200 import AdmmConfig, baseline_code, decode_batch

    code = baseline_code("cfg1_n96")
    with pytest.raises(RuntimeError):
        decode_batch(np.zeros((1, 96)), code, AdmmConfig(), want_state=True, engine=engine)


@pytest.mark.parametrize("engine", ["auto", "streaming", "wide"])
def test_fused_synthesis_equals_materialised_llrs(cuda_ok, engine):
    """decode_synth (LLRs generated inside the decode kernel) == decode_batch
    on the LLRs synth_llr writes out; trial-indexed, so any split agrees."""
    from paper_1204_0556_b200 import AdmmConfig, Awgn, Bsc, baseline_code, decode_batch, decode_synth, synth_llr

    code = baseline_code("cfg2_n1008")
    cfg = AdmmConfig(mu=5.0)
    for ch in (Awgn(2.25, code.design_rate), Bsc(0.04)):
        for dt in (torch.float32, torch.float64):
            a = decode_synth(code, ch, cfg, seed=7, point=3, trial0=100, batch=96, dtype=dt, want_x=True,
                             engine=engine)
            g = synth_llr(code.n_vars, ch, seed=7, point=3, trial0=100, batch=96, dtype=dt)
            b = decode_batch(g, code, cfg, dtype=dt, engine=engine)
            assert torch.equal(a.x, b.x) and torch.equal(a.iterations, b.iterations)
            assert torch.equal(a.flags, b.flags) and torch.equal(a.weight, b.weight)
            # shard invariance: trials 100..195 decoded as two calls
            c1 = decode_synth(code, ch, cfg, seed=7, point=3, trial0=100, batch=40, dtype=dt, engine=engine)
            c2 = decode_synth(code, ch, cfg, seed=7, point=3, trial0=140, batch=56, dtype=dt, engine=engine)
            assert torch.equal(torch.cat([c1.iterations, c2.iterations]), a.iterations)


def test_synth_llr_statistics(cuda_ok):
    from paper_1204_0556_b200 import Awgn, Bsc, synth_llr

    ch = Awgn(2.0, 0.5)
    g = synth_llr(4096, ch, seed=1, point=0, trial0=0, batch=256, dtype=torch.float64)
    var = ch.noise_variance
    y = g * var / 2.0  # received samples, mean 1, sd sqrt(var)
    assert abs(y.mean().item() - 1.0) < 0.01
    assert abs(y.std().item() - var ** 0.5) < 0.01
    b = synth_llr(4096, Bsc(0.04), seed=1, point=0, trial0=0, batch=256, dtype=torch.float64)
    frac = (b < 0).double().mean().item()
    assert abs(frac - 0.04) < 0.002
    # different points / seeds give different frames, same ones repeat exactly
    assert not torch.equal(g, synth_llr(4096, ch, seed=1, point=1, trial0=0, batch=256, dtype=torch.float64))
    assert torch.equal(g, synth_llr(4096, ch, seed=1, point=0, trial0=0, batch=256, dtype=torch.float64))


def test_phase_profiler_counts_passes(cuda_ok):
    """admm_phase_profile (tracing aid of the sharded engine) accumulates
    cycles per phase and the number of passes."""
    import ctypes

    from paper_1204_0556_b200 import AdmmConfig, Bsc, _lib, baseline_code, decode_synth

    lib = _lib.load()
    code = baseline_code("cfg5_n16384")
    _lib.check(lib.admm_phase_profile(1, None))
    r = decode_synth(code, Bsc(0.04), AdmmConfig(mu=5.0), seed=3, batch=64, dtype=torch.float32, engine="streaming")
    torch.cuda.synchronize()
    out = (ctypes.c_uint64 * 8)()
    _lib.check(lib.admm_phase_profile(0, out))
    assert r.info["engine"] == 3
    assert out[5] >= int(r.iterations.max())          # at least one pass per iteration
    assert out[0] > 0 and out[2] > 0 and out[4] > 0   # variable, check and slot phases ran


def test_wide_kernel_large_batch_matches_sharded(cuda_ok):
    """The automatic kernel choice switches to the wide HBM-streaming kernel
    for large batches on codes beyond one SM; both kernels decode the same
    trials to identical fp64 results (exact stop rule, same expression tree
    up to the residual summation order), and wide's fp32 hard decisions
    agree with fp64 on >= 99.9 % of frames."""
    from paper_1204_0556_b200 import AdmmConfig, Awgn, baseline_code, decode_synth

    code = baseline_code("cfg5_n16384")
    cfg = AdmmConfig(mu=5.0)
    ch = Awgn(2.5, code.design_rate)
    B = 2304  # > the 1024-frame switch, not a multiple of the 4096 slots
    w64 = decode_synth(code, ch, cfg, seed=1, point=1, trial0=0, batch=B, dtype=torch.float64, want_hard=True,
                       engine="streaming")
    assert w64.info["kernel"] == 5
    # the sharded kernel on a sub-batch (below the switch) of the same trials
    sub = decode_synth(code, ch, cfg, seed=1, point=1, trial0=1000, batch=200, dtype=torch.float64, want_hard=True,
                       engine="streaming")
    assert sub.info["kernel"] == 3
    # ... and the fp64 cluster engine (the automatic choice on this code)
    c64 = decode_synth(code, ch, cfg, seed=1, point=1, trial0=1000, batch=200, dtype=torch.float64, want_hard=True)
    assert c64.info["kernel_name"] == "cluster"
    assert torch.equal(c64.iterations, sub.iterations) and torch.equal(c64.hard, sub.hard)
    assert torch.equal(c64.flags, sub.flags)
    assert torch.equal(sub.iterations, w64.iterations[1000:1200])
    assert torch.equal(sub.hard, w64.hard[1000:1200])
    assert torch.equal(sub.flags, w64.flags[1000:1200])
    w32 = decode_synth(code, ch, cfg, seed=1, point=1, trial0=0, batch=B, dtype=torch.float32, want_hard=True,
                       engine="streaming")
    same = w32.hard.eq(w64.hard).all(dim=1).float().mean().item()
    assert same >= 0.999
    assert abs(int(w32.iterations.sum()) - int(w64.iterations.sum())) <= 0.02 * int(w64.iterations.sum())


@pytest.mark.parametrize("dt", [torch.float32, torch.float64])
def test_wide_direct_retirement_equals_retiring_pass(cuda_ok, dt):
    """Without per-variable outputs the wide kernel retires a converged frame
    in the pass that converged it, from the weight / integrality / syndrome
    statistics of x_t accumulated every pass; with x or hard decisions
    requested it spends a retiring pass.  Both give the same per-frame
    results (iterations, flags, weight), on AWGN and on BSC frames."""
    from paper_1204_0556_b200 import AdmmConfig, Awgn, Bsc, baseline_code, decode_synth

    code = baseline_code("cfg5_n16384")
    cfg = AdmmConfig(mu=5.0)
    for k, ch in enumerate((Awgn(2.0, code.design_rate), Bsc(0.045))):
        a = decode_synth(code, ch, cfg, seed=3, point=k, trial0=0, batch=2560, dtype=dt, engine="wide")
        b = decode_synth(code, ch, cfg, seed=3, point=k, trial0=0, batch=2560, dtype=dt, engine="wide",
                         want_hard=True)
        assert a.info["kernel"] == 5 and b.info["kernel"] == 5
        assert torch.equal(a.iterations, b.iterations)
        assert torch.equal(a.flags, b.flags)
        assert torch.equal(a.weight, b.weight)
        assert torch.equal(b.weight, b.hard.to(torch.int32).sum(dim=1))


@pytest.mark.parametrize("dt", [torch.float32, torch.float64])
def test_wide_device_llrs_match_sharded(cuda_ok, dt):
    """decode_batch on device LLRs (the fresh-slot LLRs come from the caller's
    array, not the synthesis buffer) on the wide kernel at a batch that fills
    several stripes of both stripe groups: iteration counts equal the sharded
    kernel's frame by frame, with and without per-variable outputs, and x
    after a fixed iteration count agrees to rounding."""
    from paper_1204_0556_b200 import AdmmConfig, Awgn, baseline_code, decode_batch, synth_llr

    code = baseline_code("cfg5_n16384")
    B = 2304
    g = synth_llr(code.n_vars, Awgn(2.5, code.design_rate), seed=5, point=0, trial0=0, batch=B, dtype=dt)
    cfg = AdmmConfig(mu=5.0)
    ref = torch.cat([decode_batch(g[lo:lo + 256], code, cfg, dtype=dt, want_x=False, engine="streaming").iterations
                     for lo in range(0, B, 256)])
    for want_x in (False, True):
        w = decode_batch(g, code, cfg, dtype=dt, want_x=want_x, engine="wide")
        assert w.info["kernel"] == 5
        if dt == torch.float64:
            assert torch.equal(w.iterations, ref)
        else:
            # fp32: the wide kernel keeps (z, message) and recovers lambda, a
            # different rounding from the sharded kernel's; a rare frame may
            # stop one iteration apart
            assert (w.iterations != ref).float().mean().item() <= 0.002
    fixed = AdmmConfig(mu=5.0, epsilon=1e-300, t_max=3)
    w = decode_batch(g, code, fixed, dtype=dt, engine="wide")
    r = torch.cat([decode_batch(g[lo:lo + 256], code, fixed, dtype=dt, engine="streaming").x for lo in range(0, B, 256)])
    assert (w.x - r).abs().max().item() <= (1e-5 if dt == torch.float32 else 1e-12)


@pytest.mark.parametrize("n,m,batch", [(5200, 2600, 1536), (5203, 2601, 1100)])
def test_wide_irregular_code_multi_stripe_matches_sharded(cuda_ok, n, m, batch):
    """An irregular code too large for one SM (check degrees 4-8, variable
    degrees up to 4, some of degree 0) on the generic wide kernel at a batch
    spanning both stripe groups -- also with partial variable / check blocks
    and a partial last stripe: fp64 iteration counts, flags and weights equal
    the sharded kernel's frame by frame."""
    from paper_1204_0556_b200 import AdmmConfig, ParityCheckMatrix, decode_batch

    rng = np.random.default_rng(11)
    deg = np.zeros(n, dtype=int)
    rows = []
    for c in range(m):
        d = int(rng.integers(4, 9))
        free = np.nonzero(deg < 4)[0]  # variable degrees at most 4 (the wide kernel's bucket)
        r = sorted(rng.choice(free, size=d, replace=False).tolist())
        deg[r] += 1
        rows.append(r)
    code = ParityCheckMatrix(n, rows)
    assert code.n_checks == m
    g = torch.as_tensor(rng.normal(1.2, 1.0, (batch, n)))
    cfg = AdmmConfig(mu=3.0, t_max=200)
    w = decode_batch(g, code, cfg, dtype=torch.float64, want_x=False, engine="wide")
    assert w.info["kernel"] == 5
    parts = [decode_batch(g[lo:lo + 512], code, cfg, dtype=torch.float64, want_x=False) for lo in range(0, batch, 512)]
    assert parts[0].info["kernel"] == 3
    assert torch.equal(w.iterations, torch.cat([q.iterations for q in parts]))
    assert torch.equal(w.flags, torch.cat([q.flags for q in parts]))
    assert torch.equal(w.weight, torch.cat([q.weight for q in parts]))


def test_cluster_engine_matches_wide_and_synthesis(cuda_ok):
    """Cluster engine (fp32, csrc/cluster.cuh) on config 5: identical
    decisions and iteration counts to the wide HBM kernel on the same
    synthesised frames (both fp32, same arithmetic per edge), in-kernel
    synthesis == materialised LLRs, and batch-split invariance."""
    from paper_1204_0556_b200 import AdmmConfig, Awgn, Bsc, baseline_code, decode_batch, decode_synth, synth_llr

    code = baseline_code("cfg5_n16384")
    cfg = AdmmConfig(mu=5.0)
    for k, ch in enumerate((Bsc(0.04), Awgn(2.5, code.design_rate), Awgn(1.5, code.design_rate))):
        a = decode_synth(code, ch, cfg, seed=3, point=k, trial0=50, batch=300, want_hard=True, engine="cluster")
        assert a.info["kernel_name"] == "cluster"
        w = decode_synth(code, ch, cfg, seed=3, point=k, trial0=50, batch=300, want_hard=True, engine="wide")
        same = (a.hard == w.hard).all(dim=1).float().mean().item()
        assert same >= 0.99, same
        assert (a.iterations - w.iterations).abs().float().mean().item() <= 0.05 * max(1.0, w.iterations.float().mean().item())
        g = synth_llr(code.n_vars, ch, seed=3, point=k, trial0=50, batch=300, dtype=torch.float32)
        b = decode_batch(g, code, cfg, dtype=torch.float32, want_hard=True, engine="cluster")
        assert torch.equal(a.hard, b.hard) and torch.equal(a.iterations, b.iterations)
        assert torch.equal(a.flags, b.flags) and torch.equal(a.weight, b.weight)
        c1 = decode_synth(code, ch, cfg, seed=3, point=k, trial0=50, batch=17, engine="cluster")
        assert torch.equal(c1.iterations, a.iterations[:17])


def test_cluster_sizes_agree(cuda_ok, monkeypatch):
    """The default 8-CTA clusters (two CTAs per SM) and the 4-CTA fallback
    decode every frame identically: the partition changes which CTA owns a
    check, not the arithmetic of any edge or the (exact) stop rule."""
    import copy

    from paper_1204_0556_b200 import AdmmConfig, Awgn, baseline_code, decode_synth

    code = baseline_code("cfg5_n16384")
    cfg = AdmmConfig(mu=5.0)
    ch = Awgn(2.0, code.design_rate)
    a = decode_synth(code, ch, cfg, seed=11, point=0, trial0=7, batch=96, want_hard=True, engine="cluster")
    assert a.info["cluster_size"] == 8 and a.info["cluster_threads"] == 512
    monkeypatch.setenv("ADMM_B200_CLUSTER", "4")
    code4 = copy.copy(code)
    code4._device_graphs = {}
    b = decode_synth(code4, ch, cfg, seed=11, point=0, trial0=7, batch=96, want_hard=True, engine="cluster")
    assert b.info["cluster_size"] == 4 and b.info["cluster_threads"] == 1024
    assert torch.equal(a.iterations, b.iterations) and torch.equal(a.flags, b.flags)
    assert torch.equal(a.hard, b.hard) and torch.equal(a.weight, b.weight)


def test_cluster_engine_fp64_and_state_io(cuda_ok, monkeypatch):
    import copy

    from paper_1204_0556_b200 import AdmmConfig, baseline_code, decode_batch

    code = baseline_code("cfg5_n16384")
    g = np.full((2, code.n_vars), 3.0)
    r = decode_batch(g, code, AdmmConfig(), dtype=torch.float64, engine="cluster")
    assert r.info["kernel_name"] == "cluster" and bool(r.converged.all())
    for dt in (torch.float32, torch.float64):  # state I/O goes through the step API at this size
        with pytest.raises(RuntimeError):
            decode_batch(g, code, AdmmConfig(), dtype=dt, want_state=True, engine="cluster")
    # 4-CTA clusters have no room for the fp64 state: explicit requests are refused, auto streams
    monkeypatch.setenv("ADMM_B200_CLUSTER", "4")
    code4 = copy.copy(code)
    code4._device_graphs = {}
    with pytest.raises(RuntimeError):
        decode_batch(g, code4, AdmmConfig(), dtype=torch.float64, engine="cluster")
    r = decode_batch(g, code4, AdmmConfig(), dtype=torch.float64)
    assert r.info["kernel_name"] in ("sharded", "wide") and bool(r.converged.all())


def test_config5_large_batch_properties(cuda_ok):
    """At bench scale the oracle cannot follow, so size-independent properties
    stand in: 131,072 config-5 frames per point decoded in one launch equal
    the same trials decoded in uneven pieces (a frame's result depends only
    on its trial index), every frame converges to the transmitted all-zero
    codeword with its ML certificate at these channel points, and fp32 and
    fp64 agree on every hard decision of a 4,096-frame sub-block."""
    from paper_1204_0556_b200 import AdmmConfig, Awgn, Bsc, baseline_code, decode_synth

    code = baseline_code("cfg5_n16384")
    cfg = AdmmConfig(mu=5.0)
    B = 131072
    for k, ch in enumerate((Bsc(0.04), Awgn(2.5, code.design_rate))):
        a = decode_synth(code, ch, cfg, seed=1, point=k, trial0=0, batch=B)
        assert a.info["kernel_name"] == "cluster"
        cuts = [0, 7, 4096 + 13, 70001, B]
        parts = [decode_synth(code, ch, cfg, seed=1, point=k, trial0=lo, batch=hi - lo) for lo, hi in zip(cuts, cuts[1:])]
        assert torch.equal(a.iterations, torch.cat([q.iterations for q in parts]))
        assert torch.equal(a.flags, torch.cat([q.flags for q in parts]))
        assert torch.equal(a.weight, torch.cat([q.weight for q in parts]))
        assert bool(a.converged.all()) and bool(a.codeword.all()) and int(a.weight.sum()) == 0
        assert int(a.iterations.max()) < cfg.t_max
        h32 = decode_synth(code, ch, cfg, seed=1, point=k, trial0=50000, batch=4096, want_hard=True)
        h64 = decode_synth(code, ch, cfg, seed=1, point=k, trial0=50000, batch=4096, want_hard=True, dtype=torch.float64)
        assert torch.equal(h32.hard, h64.hard)
        assert torch.equal(h32.iterations, a.iterations[50000:54096])
        assert (h32.iterations - h64.iterations).abs().float().mean().item() <= 0.05
