"""Exercise every CUDA kernel of libadmm_b200.so on small shapes, for
compute-sanitizer (racecheck / synccheck / memcheck / initcheck):

    compute-sanitizer --tool racecheck python tools/sanitize.py [kernel ...]

kernels: regular generic f64regular sharded wide cluster bp steps project.
Small codes keep the instrumented runs short; every engine is forced onto a
code it can decode (the streaming, wide and cluster engines run any code
they fit).  Results are checked against each other so a silent corruption
under instrumentation also fails.
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1204_0556_b200 as P  # noqa: E402

print("library", P._lib.load()._name, "build flags", P._lib.load().admm_build_flags(), flush=True)
which = set(sys.argv[1:]) or {"regular", "generic", "f64regular", "sharded", "wide", "cluster", "bp", "steps", "project"}
cfg = P.AdmmConfig(mu=5.0, t_max=200)
c1 = P.baseline_code("cfg1_n96")
c2 = P.baseline_code("cfg2_n1008")
g1 = P.trial_gammas(96, P.Awgn(2.5, 0.5), 1, 0, range(8))
ref = P.decode_batch(g1, c1, cfg, dtype=torch.float64, want_hard=True)
torch.cuda.synchronize()


def same(res, tag):
    torch.cuda.synchronize()
    agree = (res.hard.cpu() == ref.hard.cpu()).all(dim=1).float().mean().item()
    print(f"{tag}: kernel {res.info.get('kernel_name')}, hard decisions agree on {agree:.2f} of frames", flush=True)
    assert agree >= 0.85, tag


if "regular" in which:
    same(P.decode_batch(g1, c1, cfg, dtype=torch.float32, want_hard=True), "resident regular fp32")
if "f64regular" in which:
    same(ref, "resident regular fp64")
if "generic" in which:
    irr = P.ParityCheckMatrix(12, [list(range(0, 8)), list(range(4, 11)), [0, 7, 10]])
    gi = np.random.default_rng(4).normal(0.5, 1.2, (6, 12))
    for dt in (torch.float32, torch.float64):
        r = P.decode_batch(gi, irr, cfg, dtype=dt)
        torch.cuda.synchronize()
        print("resident generic", dt, r.info["kernel_name"], r.iterations.tolist(), flush=True)
if "sharded" in which:
    for dt in (torch.float32, torch.float64):
        same(P.decode_batch(g1, c1, cfg, dtype=dt, want_hard=True, engine="streaming"), f"sharded {dt}")
if "wide" in which:
    for dt in (torch.float32, torch.float64):
        same(P.decode_batch(g1, c1, cfg, dtype=dt, want_hard=True, engine="wide"), f"wide {dt}")
        s = P.decode_synth(c1, P.Awgn(2.5, 0.5), cfg, seed=1, point=0, trial0=0, batch=8, dtype=dt, engine="wide")
        torch.cuda.synchronize()
        print(f"wide synth {dt}", s.iterations.tolist(), flush=True)
if "cluster" in which:
    g2 = P.trial_gammas(1008, P.Awgn(2.5, 0.5), 1, 0, range(6))
    a = P.decode_batch(g2, c2, cfg, dtype=torch.float32, want_hard=True, engine="cluster")
    b = P.decode_batch(g2, c2, cfg, dtype=torch.float64, want_hard=True)
    torch.cuda.synchronize()
    agree = (a.hard.cpu() == b.hard.cpu()).all(dim=1).float().mean().item()
    print(f"cluster fp32 (config-2 code, {a.info['cluster_size']} CTAs): kernel {a.info['kernel_name']}, "
          f"agree with fp64 {agree:.2f}", flush=True)
    assert a.info["kernel_name"] == "cluster" and agree >= 0.8
    s = P.decode_synth(c2, P.Bsc(0.04), cfg, seed=2, point=0, trial0=0, batch=6, engine="cluster")
    torch.cuda.synchronize()
    print("cluster synth iterations", s.iterations.tolist(), flush=True)
    c = P.decode_batch(g2, c2, cfg, dtype=torch.float64, want_hard=True, engine="cluster")
    torch.cuda.synchronize()
    print(f"cluster fp64: kernel {c.info['kernel_name']}, iterations equal to the resident fp64 kernel: "
          f"{torch.equal(c.iterations, b.iterations)}", flush=True)
    assert c.info["kernel_name"] == "cluster" and torch.equal(c.iterations, b.iterations) and torch.equal(c.hard, b.hard)
if "bp" in which:
    r = P.decode_bp_batch(g1, c1, P.BpConfig(t_max=30), dtype=torch.float64)
    torch.cuda.synchronize()
    print("bp", r.iterations.tolist(), flush=True)
if "steps" in which:
    st = P.AdmmState.initial(c1, batch=4, device="cuda")
    gg = torch.as_tensor(g1[:4], device="cuda")
    for _ in range(3):
        P.x_update(st, c1, gg, cfg)
        P.z_update(st, c1, cfg)
        P.lambda_update(st, c1, cfg)
    print("steps ok", float(st.x.sum()), flush=True)
    print("membership", P.membership_batch(np.random.default_rng(0).uniform(-0.1, 1.1, (64, 6))).sum(), flush=True)
if "project" in which:
    z = P.project_batch(np.random.default_rng(1).uniform(-1, 2, (100, 13)))
    lv = P.synth_llr(96, P.Bsc(0.04), seed=1, point=0, trial0=0, batch=4)
    torch.cuda.synchronize()
    print("project / synth ok", z.shape, tuple(lv.shape), flush=True)
print("SANITIZE-DONE", sorted(which))
