"""One decode call for profiling (ncu -k regex:resident -c 1 python tools/prof_decode.py ...).

Decodes --frames synthetic AWGN frames of a BASELINE code at one SNR after a
warm-up call, so an ncu capture sees exactly one steady-state launch.
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1204_0556_b200 import AdmmConfig, Awgn, baseline_code, decode_batch, synth_llr  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--code", default="cfg2_n1008")
ap.add_argument("--frames", type=int, default=8192)
ap.add_argument("--snr", type=float, default=1.5)
ap.add_argument("--dtype", choices=["f32", "f64"], default="f32")
a = ap.parse_args()
dt = torch.float32 if a.dtype == "f32" else torch.float64
code = baseline_code(a.code)
g = synth_llr(code.n_vars, Awgn(a.snr, code.design_rate), seed=5, point=0, trial0=0, batch=a.frames, dtype=dt)
cfg = AdmmConfig(mu=5.0)
decode_batch(g[:256], code, cfg, dtype=dt, want_x=False)
torch.cuda.synchronize()
r = decode_batch(g, code, cfg, dtype=dt, want_x=False)
torch.cuda.synchronize()
print("frames", a.frames, "mean iterations", r.iterations.float().mean().item())
