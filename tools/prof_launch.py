"""Exactly one decode launch of a bench.py workload, for ncu.

    ncu --set full -k regex:wide -c 1 python tools/prof_launch.py --workload cfg5 --frames 262144

Runs a 256-frame warm-up call first (builds the device graph; on codes
beyond one SM it runs the sharded kernel, so a `-k regex:` filter on the
main kernel sees only the measured launch), then the launch bench.py times:
cfg5 -> decode_synth of point 0 (BSC 0.04), trials [0, frames); cfg1-4 ->
decode_batch of device LLRs of point 0.  Prints one JSON line with the
launch's edge-updates, so ncu's per-launch DRAM bytes and instruction count
can be normalised per edge-update (profiles/traffic.json).
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1204_0556_b200 import AdmmConfig, baseline_code, decode_batch, decode_synth  # noqa: E402
from paper_1204_0556_b200.channels import awgn_gammas_device, bsc_gammas_device  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="cfg5", choices=sorted(bench.WORKLOADS))
ap.add_argument("--frames", type=int, default=0)
ap.add_argument("--dtype", choices=["f32", "f64"], default="f32")
a = ap.parse_args()
wl = bench.WORKLOADS[a.workload]
dt = torch.float32 if a.dtype == "f32" else torch.float64
code = baseline_code(wl.code)
cfg = AdmmConfig(mu=bench.MU, epsilon=bench.EPS, t_max=bench.TMAX, rho=bench.RHO)
F = a.frames or (262144 if wl.source == "synth" else wl.frames)
kind, val = wl.points[0]
ch = bench.channel_of(wl.points[0], code)
if wl.source == "synth":
    decode_synth(code, ch, cfg, seed=1, point=0, trial0=0, batch=256, dtype=dt)
    torch.cuda.synchronize()
    r = decode_synth(code, ch, cfg, seed=1, point=0, trial0=0, batch=F, dtype=dt)
else:
    seed = 1000003
    g = (bsc_gammas_device(F, code.n_vars, val, seed=seed, dtype=dt) if kind == "bsc" else
         awgn_gammas_device(F, code.n_vars, val, code.design_rate, seed=seed, dtype=dt))
    decode_batch(g[:256], code, cfg, dtype=dt, want_x=False, validate=False)
    torch.cuda.synchronize()
    r = decode_batch(g, code, cfg, dtype=dt, want_x=False, validate=False)
torch.cuda.synchronize()
it = int(r.iterations.to(torch.int64).sum())
print(json.dumps({"workload": a.workload, "dtype": a.dtype, "frames": F, "kernel": r.info["kernel"],
                  "kernel_name": r.info["kernel_name"], "iterations": it, "edge_updates": it * code.n_edges}))
