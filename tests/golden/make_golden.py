"""Generate the golden fixtures in tests/golden/ from the REFERENCE package.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

Everything stored here is an output of the read-only reference
``polylp`` (/root/reference/pkg/src/polylp) on seeded inputs; the oracle
(oracle/admm_oracle.py) and the CUDA path are both checked against these
files, and neither the GPU tests nor bench.py read /root/reference.

Fixtures
--------
projection.npz     project_batch on adversarial rows for d = 1..13 plus the
                   reference's KAT rows (test_parity_polytope.py:139-157).
decode_cfg1.npz    BASELINE config 1: (3,6) n=96 from make_ldpc(seed 0,
                   parallel edges repaired), AWGN 3.0 dB, frames
                   trial_gamma(seed=1, point=0, trial=t) for t < 1000,
                   AdmmConfig(mu=5.0): iterations, status, hard decisions,
                   integral, certificate for all 1000 frames, full x for the
                   first 200.
fixed_cfg1.npz     config-1 frames 0..15 decoded for a FIXED number of
                   iterations (epsilon=1e-300 so eps^2 == 0) T = 1, 50, 1000.
decode_cfg2.npz    config-2 code (n=1008, girth 6) at 2.0 dB, 24 frames.
decode_cfg4.npz    config-4 code ((3,13), n=1040, girth 6) at 4.0 dB, 24 frames.
harness.npz        reference sweep()/run_point() CSV (timing=False) on the config-1
                   code: fixed-count sweep over BSC 0.03 / AWGN 2.5 dB and a
                   target-errors run (exact truncation), for the GPU harness.
steps.npz          single-iteration state dumps (x, z, lam) after 1, 2, 3
                   iterations for one config-1 frame (x_update / z_update /
                   lambda_update driven directly, as test_admm.py:151-160).
sweep_*.npz        sweep END POINTS of the BASELINE workloads (round 2): for each
                   (config, channel point) 1000 frames (256 for config 5)
                   trial_gamma(seed=1, point=k, trial=t), AdmmConfig(mu=5.0):
                   iterations, status, integral, certificate, packed hard
                   decisions, x of the first frames.  Points: cfg2 1.5 / 3.0 dB,
                   cfg3 1.5 / 2.0 / 3.0 dB, cfg4 3.5 / 5.0 dB, cfg5 BSC 0.04 /
                   AWGN 2.5 dB.  Decoded over a process pool (`sweep`).
conformance.npz    the reference's decode properties and acceptance criteria
                   5-7 as data (`conformance`): Hamming one-flip LP values and
                   ML words (test_admm.py:116-135), the codebook certificate
                   case (:170-184), LP value of the objective case (:186-197),
                   the feasibility case's final z (:147-168), criterion 5/6
                   iteration counts and the criterion 7 WERs
                   (test_acceptance.py:186-262).
membership.npz     membership() on adversarial rows d = 1..10 (inside, outside,
                   boundary, projected points) (parity_polytope.py:69-91).
bp.npz             the reference's BP (bp_decoder.py): config-1 code at 2.5 dB,
                   200 frames with the default BpConfig (beliefs, iterations,
                   found, decode_bp x / integral / status), 16 frames for a
                   FIXED 1 / 5 / 30 iterations (early_stop=False); a mixed-degree
                   code; 25 random tree codes (the reference's
                   tests/oracles.py:random_tree_code, seed 0) with their
                   exact marginals (oracles.exact_marginals) and the BP beliefs
                   after 40 iterations at llr_clip=500 (test_bp.py:31-42);
                   config-2 code at 1.75 dB, 24 frames (iterations, found, hard).
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

import polylp  # noqa: E402  (the reference, read-only)
from polylp import AdmmConfig, decode, project_batch  # noqa: E402
from polylp.admm_decoder import AdmmState, lambda_update, x_update, z_update  # noqa: E402

from paper_1204_0556_b200.codes import baseline_code  # noqa: E402

OUT = Path(__file__).resolve().parent


def ref_code(code):
    return polylp.ParityCheckMatrix(code.n_vars, [np.asarray(c) for c in code.check_neighborhoods])


def pack_checks(code):
    return code.check_ptr.astype(np.int64), code.edge_var.astype(np.int64)


def awgn_frames(code, snr_db, seed, point, trials):
    ch = polylp.Awgn(snr_db, code.design_rate)
    out = []
    for t in trials:
        rng = np.random.default_rng(np.random.SeedSequence(entropy=seed, spawn_key=(point, t)))
        y = polylp.transmit(np.zeros(code.n_vars, dtype=np.uint8), ch, rng)
        out.append(polylp.llr(y, ch))
    return np.array(out)


def projection_fixture():
    rng = np.random.default_rng(20241020)
    rec = {}
    for d in range(1, 14):
        rows = np.concatenate([
            rng.uniform(-2.0, 3.0, size=(160, d)),
            rng.integers(-1, 3, size=(40, d)).astype(float),       # exact ties at 0 / 1
            np.round(rng.uniform(-1.0, 2.0, size=(40, d)) * 4) / 4,  # quarter grid
            rng.normal(0.5, 0.6, size=(80, d)),
        ])
        rec[f"in_d{d}"] = rows
        rec[f"out_d{d}"] = project_batch(rows)
    kat_in = [[1, 1, 0, 0], [1, 0, 0], [1, -0.2], [0, 0, 1], [0.7], [-3.0]]
    for k, u in enumerate(kat_in):
        u = np.array([u], dtype=float)
        rec[f"kat_in_{k}"] = u
        rec[f"kat_out_{k}"] = project_batch(u)
    np.savez_compressed(OUT / "projection.npz", **rec)


def decode_fixture(name, code, snr_db, n_frames, n_x, cfg):
    rc = ref_code(code)
    gam = awgn_frames(code, snr_db, seed=1, point=0, trials=range(n_frames))
    iters = np.zeros(n_frames, np.int32)
    status = np.zeros(n_frames, np.uint8)
    integral = np.zeros(n_frames, np.uint8)
    cert = np.zeros(n_frames, np.uint8)
    hard = np.zeros((n_frames, code.n_vars), np.uint8)
    xs = np.zeros((n_x, code.n_vars))
    for t in range(n_frames):
        out = decode(gam[t], rc, cfg)
        iters[t] = out.iterations
        status[t] = out.status == polylp.STATUS_CONVERGED
        integral[t] = out.integral
        cert[t] = out.ml_certificate
        hard[t] = out.hard_decision
        if t < n_x:
            xs[t] = out.x
    ptr, ev = pack_checks(code)
    np.savez_compressed(
        OUT / name, n_vars=code.n_vars, check_ptr=ptr, edge_var=ev, snr_db=snr_db,
        mu=cfg.mu, epsilon=cfg.epsilon, t_max=cfg.t_max, rho=cfg.rho,
        gamma_head=gam[:n_x], iterations=iters, converged=status, integral=integral,
        certificate=cert, hard=np.packbits(hard, axis=1), x=xs)
    print(name, "mean iters", iters.mean(), "word errors", int((hard.sum(1) > 0).sum()))


def fixed_fixture(code):
    rc = ref_code(code)
    gam = awgn_frames(code, 3.0, seed=1, point=0, trials=range(16))
    rec = {"gamma": gam}
    for T in (1, 50, 1000):
        cfg = AdmmConfig(mu=5.0, epsilon=1e-300, t_max=T)
        rec[f"x_T{T}"] = np.array([decode(g, rc, cfg).x for g in gam])
    ptr, ev = pack_checks(code)
    np.savez_compressed(OUT / "fixed_cfg1.npz", n_vars=code.n_vars, check_ptr=ptr, edge_var=ev, **rec)


def steps_fixture(code):
    rc = ref_code(code)
    gam = awgn_frames(code, 3.0, seed=1, point=0, trials=[7])[0]
    cfg = AdmmConfig(mu=5.0)
    st = AdmmState.initial(rc)
    rec = {"gamma": gam}
    for t in range(1, 4):
        x_update(st, rc, gam, cfg)
        z_update(st, rc, cfg)
        lambda_update(st, rc, cfg)
        rec[f"x{t}"] = st.x.copy()
        rec[f"z{t}"] = st.z.copy()
        rec[f"lam{t}"] = st.lam.copy()
    ptr, ev = pack_checks(code)
    np.savez_compressed(OUT / "steps.npz", n_vars=code.n_vars, check_ptr=ptr, edge_var=ev, **rec)


def harness_fixture(code):
    from polylp import Awgn, Bsc, DecoderRef, run_point, stats_to_csv, sweep

    rc = ref_code(code)
    dec = DecoderRef("admm", AdmmConfig(mu=3.0))
    csv_sweep = stats_to_csv(sweep(rc, [Bsc(0.03), Awgn(2.5, rc.design_rate)], dec, n_trials=300, seed=107,
                                   workers=1), timing=False)
    csv_target = stats_to_csv([run_point(rc, Bsc(0.05), dec, target_errors=20, max_trials=5000, seed=108,
                                         point_index=2)], timing=False)
    ptr, ev = pack_checks(code)
    np.savez_compressed(OUT / "harness.npz", n_vars=code.n_vars, check_ptr=ptr, edge_var=ev,
                        csv_sweep=np.array(csv_sweep), csv_target=np.array(csv_target))
    print(csv_sweep, csv_target)


def bp_fixture():
    from polylp import BpConfig, decode_bp, posterior_llrs

    sys.path.insert(0, "/root/reference/pkg/tests")
    import oracles  # noqa: E402  (the reference's own test oracles)

    rec = {}
    c1 = baseline_code("cfg1_n96")
    rc = ref_code(c1)
    gam = awgn_frames(c1, 2.5, seed=1, point=0, trials=range(200))
    bel, it, fd, xs, integ, stat = [], [], [], [], [], []
    for g in gam:
        b, t, f = posterior_llrs(g, rc, BpConfig())
        o = decode_bp(g, rc, BpConfig())
        bel.append(b); it.append(t); fd.append(f); xs.append(o.x); integ.append(o.integral)
        stat.append(o.status == polylp.STATUS_CONVERGED)
    ptr, ev = pack_checks(c1)
    rec.update(c1_check_ptr=ptr, c1_edge_var=ev, c1_n_vars=c1.n_vars, c1_gamma=gam, c1_beliefs=np.array(bel),
               c1_iterations=np.array(it), c1_found=np.array(fd), c1_x=np.array(xs), c1_integral=np.array(integ),
               c1_status=np.array(stat))
    for T in (1, 5, 30):
        rec[f"c1_fixed_T{T}"] = np.array([posterior_llrs(g, rc, BpConfig(t_max=T, early_stop=False))[0]
                                          for g in gam[:16]])
    # mixed check degrees (2 .. 7) and a degree-1 variable
    rng = np.random.default_rng(77)
    mixed = [sorted(rng.choice(40, size=int(rng.integers(2, 8)), replace=False).tolist()) for _ in range(22)]
    mcode = polylp.ParityCheckMatrix(40, [np.array(c) for c in mixed])
    mg = rng.normal(0.8, 1.3, size=(12, 40))
    rec["mx_checks"] = np.array([len(c) for c in mixed])
    rec["mx_flat"] = np.concatenate(mixed)
    rec["mx_gamma"] = mg
    rec["mx_beliefs_T7"] = np.array([posterior_llrs(g, mcode, BpConfig(t_max=7, early_stop=False, llr_clip=12.0))[0]
                                     for g in mg])
    out = [posterior_llrs(g, mcode, BpConfig(t_max=60)) for g in mg]
    rec["mx_beliefs"] = np.array([o[0] for o in out])
    rec["mx_iterations"] = np.array([o[1] for o in out])
    rec["mx_found"] = np.array([o[2] for o in out])
    # tree codes: BP is exact (test_bp.py:31-42)
    trng = np.random.default_rng(0)
    for k in range(25):
        tc = oracles.random_tree_code(trng, n_max=12)
        g = trng.normal(0.0, 1.5, tc.n_vars)
        b, _, _ = posterior_llrs(g, tc, BpConfig(t_max=40, llr_clip=500.0, early_stop=False))
        rec[f"tree{k}_n"] = tc.n_vars
        rec[f"tree{k}_lens"] = np.array([len(c) for c in tc.check_neighborhoods])
        rec[f"tree{k}_flat"] = np.concatenate([np.asarray(c) for c in tc.check_neighborhoods])
        rec[f"tree{k}_gamma"] = g
        rec[f"tree{k}_beliefs"] = b
        rec[f"tree{k}_exact"] = oracles.exact_marginals(g, tc)
    c2 = baseline_code("cfg2_n1008")
    rc2 = ref_code(c2)
    g2 = awgn_frames(c2, 1.75, seed=1, point=0, trials=range(24))
    o2 = [decode_bp(g, rc2, BpConfig(t_max=200)) for g in g2]
    rec.update(c2_gamma=g2, c2_iterations=np.array([o.iterations for o in o2]),
               c2_found=np.array([o.status == polylp.STATUS_CONVERGED for o in o2]),
               c2_hard=np.packbits(np.array([o.hard_decision for o in o2]), axis=1))
    from polylp import Bsc, DecoderRef, stats_to_csv, sweep

    rec["c1_csv_bp"] = np.array(stats_to_csv(sweep(rc, [Bsc(0.04), polylp.Awgn(2.0, rc.design_rate)],
                                                   DecoderRef("bp", BpConfig(t_max=100)), n_trials=200,
                                                   seed=109, workers=1), timing=False))
    np.savez_compressed(OUT / "bp.npz", **rec)
    print("bp: cfg1 mean iters", np.mean(it), "found", int(np.sum(fd)), "cfg2 found",
          int(rec["c2_found"].sum()), "iters", rec["c2_iterations"])


# ---------------------------------------------------------------------------
# Round 2: sweep end points, conformance properties, membership
# ---------------------------------------------------------------------------
SWEEP_POINTS = [
    # (fixture name, baseline code, channel, channel parameter, point index, frames, frames with x)
    ("sweep_cfg2_1p5.npz", "cfg2_n1008", "awgn", 1.5, 0, 1000, 16),
    ("sweep_cfg2_3p0.npz", "cfg2_n1008", "awgn", 3.0, 6, 1000, 16),
    ("sweep_cfg3_1p5.npz", "cfg3_n2640", "awgn", 1.5, 3, 1000, 16),
    ("sweep_cfg3_2p0.npz", "cfg3_n2640", "awgn", 2.0, 0, 1000, 16),
    ("sweep_cfg3_3p0.npz", "cfg3_n2640", "awgn", 3.0, 2, 1000, 16),
    ("sweep_cfg4_3p5.npz", "cfg4_n1040", "awgn", 3.5, 0, 1000, 16),
    ("sweep_cfg4_5p0.npz", "cfg4_n1040", "awgn", 5.0, 3, 1000, 16),
    ("sweep_cfg5_bsc.npz", "cfg5_n16384", "bsc", 0.04, 0, 256, 8),
    ("sweep_cfg5_awgn.npz", "cfg5_n16384", "awgn", 2.5, 1, 256, 8),
]


def _channel(code, kind, val):
    return polylp.Bsc(val) if kind == "bsc" else polylp.Awgn(val, code.design_rate)


def _sweep_chunk(args):
    n_vars, checks, kind, val, point, trials, n_x = args
    rc = polylp.ParityCheckMatrix(n_vars, [np.asarray(c) for c in checks])
    ch = _channel(rc, kind, val)
    cfg = AdmmConfig(mu=5.0)
    out = []
    for t in trials:
        rng = np.random.default_rng(np.random.SeedSequence(entropy=1, spawn_key=(point, t)))
        g = polylp.llr(polylp.transmit(np.zeros(n_vars, dtype=np.uint8), ch, rng), ch)
        o = decode(g, rc, cfg)
        out.append((t, o.iterations, o.status == polylp.STATUS_CONVERGED, o.integral, o.ml_certificate,
                    np.packbits(o.hard_decision), o.x if t < n_x else None))
    return out


def sweep_fixtures(only=None, workers=8):
    from multiprocessing import Pool

    for name, key, kind, val, point, frames, n_x in SWEEP_POINTS:
        if only and name not in only:
            continue
        code = baseline_code(key)
        checks = [np.asarray(c) for c in code.check_neighborhoods]
        # small chunks first-come: the slow (T_max) frames spread over the pool
        jobs = [(code.n_vars, checks, kind, val, point, range(lo, min(lo + 8, frames)), n_x)
                for lo in range(0, frames, 8)]
        with Pool(workers) as pool:
            recs = sorted(r for part in pool.imap_unordered(_sweep_chunk, jobs) for r in part)
        assert [r[0] for r in recs] == list(range(frames))
        ptr, ev = pack_checks(code)
        np.savez_compressed(
            OUT / name, code=key, n_vars=code.n_vars, check_ptr=ptr, edge_var=ev, channel=kind, param=val,
            point=point, seed=1, mu=5.0, epsilon=1e-5, t_max=1000, rho=1.9,
            iterations=np.array([r[1] for r in recs], np.int32), converged=np.array([r[2] for r in recs], np.uint8),
            integral=np.array([r[3] for r in recs], np.uint8), certificate=np.array([r[4] for r in recs], np.uint8),
            hard=np.stack([r[5] for r in recs]), x=np.stack([r[6] for r in recs[:n_x]]))
        it = np.array([r[1] for r in recs])
        we = sum(int(np.unpackbits(r[5]).any()) for r in recs)
        print(name, "mean iters", it.mean(), "at T_max", int((it == 1000).sum()), "word errors", we, flush=True)


def conformance_fixture():
    """The reference's decode properties and acceptance criteria 5-7 as data
    (the GPU box has no /root/reference)."""
    from polylp import Bsc, DecoderRef, gen_regular_ldpc, is_codeword, llr, run_point
    from polylp.admm_decoder import AdmmState, lambda_update, x_update, z_update

    sys.path.insert(0, "/root/reference/pkg/tests")
    import oracles  # noqa: E402  (the reference's own test oracles)

    rec = {}
    # Hamming one-flip cases (test_admm.py:116-135)
    ham = oracles.hamming_7_4()
    book = oracles.codebook(ham.to_dense())
    rec["ham_checks"] = np.concatenate([np.asarray(c) for c in ham.check_neighborhoods])
    rec["ham_check_len"] = np.array([len(c) for c in ham.check_neighborhoods])
    gam, lpv, ml, xs = [], [], [], []
    for flip in [None, 0, 1, 2, 3, 4, 5, 6]:
        y = np.zeros(7, dtype=np.uint8)
        if flip is not None:
            y[flip] = 1
        g = llr(y, Bsc(0.05))
        gam.append(g)
        lpv.append(oracles.fundamental_lp(g, ham)[0])
        ml.append(book[np.argmin(book @ g)])
        xs.append(decode(g, ham).x)
    rec.update(ham_gamma=np.array(gam), ham_lp=np.array(lpv), ham_ml=np.array(ml), ham_x=np.array(xs),
               ham_var_deg=np.asarray(ham.var_degrees))
    # ML certificate against the codebook (test_admm.py:170-184)
    c16 = gen_regular_ldpc(16, 3, 6, seed=9)
    book16 = oracles.codebook(c16.to_dense())
    rng = np.random.default_rng(2)
    g16 = []
    for _ in range(200):
        y = (rng.random(16) < 0.05).astype(np.uint8)
        g16.append(llr(y, Bsc(0.05)))
    g16 = np.array(g16)
    o16 = [decode(g, c16) for g in g16]
    rec.update(c16_book=book16, c16_gamma=g16, c16_best=(g16 @ book16.T).min(axis=1),
               c16_iterations=np.array([o.iterations for o in o16]),
               c16_cert=np.array([o.integral and is_codeword(c16, o.hard_decision) for o in o16]))
    # objective approaches the LP value (test_admm.py:186-197)
    c24 = gen_regular_ldpc(24, 3, 6, seed=3)
    g24 = np.random.default_rng(5).normal(0.4, 1.0, 24)
    rec.update(lp24_gamma=g24, lp24_value=oracles.fundamental_lp(g24, c24)[0],
               lp24_x100=decode(g24, c24, AdmmConfig(epsilon=1e-14, t_max=100, rho=1.0)).x,
               lp24_x1000=decode(g24, c24, AdmmConfig(epsilon=1e-14, t_max=1000, rho=1.0)).x)
    # feasibility at convergence (test_admm.py:147-168): final z, lambda of the reference
    c48 = gen_regular_ldpc(48, 3, 6, seed=4)
    g48 = np.random.default_rng(1).normal(0.8, 1.0, 48)
    cfg = AdmmConfig()
    st = AdmmState.initial(c48)
    thr = cfg.epsilon ** 2 * c48.n_edges
    for t in range(cfg.t_max):
        x_update(st, c48, g48, cfg)
        z_update(st, c48, cfg)
        gx = st.x[c48.edge_var]
        primal = float(((gx - st.z) ** 2).sum())
        moved = float(((st.z - st.z_prev) ** 2).sum())
        lambda_update(st, c48, cfg)
        if primal < thr and moved < thr:
            break
    rec.update(feas_gamma=g48, feas_iterations=t + 1, feas_z=st.z, feas_x=st.x)
    # acceptance criteria 5 and 6 (test_acceptance.py:186-223): per-trial iterations
    c96 = gen_regular_ldpc(96, 3, 6, seed=5)

    def tg(code, ch, seed, point, trial):
        r = np.random.default_rng(np.random.SeedSequence(entropy=seed, spawn_key=(point, trial)))
        return llr(polylp.transmit(np.zeros(code.n_vars, dtype=np.uint8), ch, r), ch)

    it5, w5 = [], []
    for t in range(2000):
        o = decode(tg(c96, Bsc(0.02), 105, 0, t), c96, AdmmConfig())
        it5.append(o.iterations)
        w5.append(int(o.hard_decision.sum()))
    it6 = {1.0: [], 1.9: []}
    for t in range(1000):
        g = tg(c96, Bsc(0.02), 106, 0, t)
        for rho in it6:
            it6[rho].append(decode(g, c96, AdmmConfig(rho=rho)).iterations)
    rec.update(crit5_iterations=np.array(it5), crit5_weight=np.array(w5), crit6_iter_rho1=np.array(it6[1.0]),
               crit6_iter_rho19=np.array(it6[1.9]))
    # criterion 7 (test_acceptance.py:226-262): WER and trials of the four runs
    c7 = {}
    for tag, cfg7, pt in (("mu3", AdmmConfig(mu=3.0), 0), ("mu7", AdmmConfig(mu=7.0), 0),
                          ("eps4", AdmmConfig(epsilon=1e-4), 1), ("eps6", AdmmConfig(epsilon=1e-6), 1)):
        s = run_point(c96, Bsc(0.03), DecoderRef("admm", cfg7), n_trials=5000, seed=107, point_index=pt, workers=8)
        c7[f"crit7_{tag}_word_errors"] = s.word_errors
        c7[f"crit7_{tag}_bit_errors"] = s.bit_errors
        c7[f"crit7_{tag}_trials"] = s.trials
    rec.update(c7)
    for name, c in (("c16", c16), ("c24", c24), ("c48", c48), ("c96", c96)):
        ptr, ev = pack_checks(c)
        rec[f"{name}_check_ptr"], rec[f"{name}_edge_var"], rec[f"{name}_n_vars"] = ptr, ev, c.n_vars
    np.savez_compressed(OUT / "conformance.npz", **rec)
    print("conformance: crit5 frac<200", float((np.array(it5)[np.array(w5) == 0] < 200).mean()),
          "crit6 ratio", sum(it6[1.9]) / sum(it6[1.0]), c7)


def membership_fixture():
    from polylp.parity_polytope import membership

    rng = np.random.default_rng(424242)
    rec = {}
    for d in range(1, 11):
        rows = [rng.uniform(-0.2, 1.2, size=(200, d)),                       # mostly outside
                project_batch(rng.uniform(-1.0, 2.0, size=(200, d))),        # on the boundary / inside
                0.5 * project_batch(rng.uniform(-1.0, 2.0, size=(100, d))) + 0.25,  # interior mixes
                rng.integers(0, 2, size=(60, d)).astype(float),              # vertices, odd ones outside
                np.round(rng.uniform(0, 1, size=(60, d)) * 4) / 4]
        rows = np.concatenate(rows)
        rec[f"in_d{d}"] = rows
        rec[f"out_d{d}"] = np.array([membership(u) for u in rows])
        rec[f"out7_d{d}"] = np.array([membership(u, 1e-7) for u in rows])
    np.savez_compressed(OUT / "membership.npz", **rec)


def main():
    projection_fixture()
    c1 = baseline_code("cfg1_n96")
    decode_fixture("decode_cfg1.npz", c1, 3.0, 1000, 200, AdmmConfig(mu=5.0))
    fixed_fixture(c1)
    steps_fixture(c1)
    harness_fixture(c1)
    decode_fixture("decode_cfg2.npz", baseline_code("cfg2_n1008"), 2.0, 24, 24, AdmmConfig(mu=5.0))
    decode_fixture("decode_cfg4.npz", baseline_code("cfg4_n1040"), 4.0, 24, 24, AdmmConfig(mu=5.0))


def main_bp():
    bp_fixture()


if __name__ == "__main__":
    if sys.argv[1:] == ["bp"]:
        main_bp()
    elif sys.argv[1:2] == ["sweep"]:
        sweep_fixtures(set(sys.argv[2:]) or None)
    elif sys.argv[1:] == ["conformance"]:
        conformance_fixture()
    elif sys.argv[1:] == ["membership"]:
        membership_fixture()
    else:
        main()
        bp_fixture()
