"""Cluster engine smoke/A-B: config-5 frames on the cluster kernel vs the wide
kernel (same synthesised frames), agreement and timing.
    python tools/cluster_check.py [--frames N]"""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1204_0556_b200 import AdmmConfig, Awgn, Bsc, baseline_code, decode_synth, device_graph  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--frames", type=int, default=4096)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
code = baseline_code("cfg5_n16384")
t0 = time.time()
dg = device_graph(code)
print("graph build %.1fs" % (time.time() - t0), dg.info, flush=True)
cfg = AdmmConfig(mu=5.0)
for k, ch in enumerate((Bsc(0.04), Awgn(2.5, 0.5))):
    res = {}
    for eng in ("auto", "wide"):
        r = decode_synth(code, ch, cfg, seed=1, point=k, trial0=0, batch=a.frames, dtype=torch.float32,
                         want_hard=True, engine=eng)
        torch.cuda.synchronize()
        ts = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            decode_synth(code, ch, cfg, seed=1, point=k, trial0=0, batch=a.frames, dtype=torch.float32, engine=eng)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        it = int(r.iterations.to(torch.int64).sum())
        ms = min(ts)
        print(f"point {k} {eng:5s} kernel={r.info['kernel_name']}: {ms:.2f} ms, {a.frames / ms * 1e3:,.0f} frames/s, "
              f"{it * code.n_edges / ms / 1e6:.1f} G eu/s, mean iters {it / a.frames:.2f}, "
              f"word errors {int((r.weight > 0).sum())}, converged {int(r.converged.sum())}", flush=True)
        res[eng] = r
    same = (res["auto"].hard == res["wide"].hard).all(dim=1).float().mean().item()
    dit = (res["auto"].iterations - res["wide"].iterations).abs().float().mean().item()
    print(f"  identical hard decisions {same:.4f}, mean |d iterations| {dit:.3f}", flush=True)
