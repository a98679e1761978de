"""BP baseline throughput on the config-2 code (device-timed, CUDA events).

    python tools/bench_bp.py [--dtype f32|f64] [--snr 2.0] [--frames 65536]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1204_0556_b200 import Awgn, BpConfig, baseline_code, decode_bp_batch, synth_llr  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dtype", choices=["f32", "f64"], default="f32")
ap.add_argument("--snr", type=float, default=2.0)
ap.add_argument("--frames", type=int, default=65536)
ap.add_argument("--t-max", type=int, default=1000)
a = ap.parse_args()
dt = torch.float32 if a.dtype == "f32" else torch.float64
code = baseline_code("cfg2_n1008")
g = synth_llr(code.n_vars, Awgn(a.snr, code.design_rate), seed=9, point=0, trial0=0, batch=a.frames, dtype=dt)
cfg = BpConfig(t_max=a.t_max)
decode_bp_batch(g[:2048], code, cfg, dtype=dt, want_beliefs=False, want_x=False)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
r = decode_bp_batch(g, code, cfg, dtype=dt, want_beliefs=False, want_x=False)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
it = r.iterations.double().sum().item()
print(f"BP {a.dtype} Eb/N0={a.snr} dB: {a.frames / ms * 1e3:,.0f} frames/s, "
      f"{it * code.n_edges / ms / 1e6:,.1f} G edge-updates/s, mean iterations {it / a.frames:.1f}, "
      f"found {r.found.float().mean().item():.4f}, info {r.info['engine']}")
