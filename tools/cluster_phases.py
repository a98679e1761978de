"""Phase split of the cluster engine's iteration (admm_cluster_phase_profile).
    python tools/cluster_phases.py [--frames N]"""
import argparse
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1204_0556_b200 import AdmmConfig, Awgn, baseline_code, decode_synth, _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--frames", type=int, default=4096)
a = ap.parse_args()
# The profiling instantiation also prints one "cta B cluster K rank R smid S"
# line per CTA: pipe the output through `grep ^cta` to see which CTAs share an
# SM (8-CTA clusters: two CTAs per SM, never of the same cluster).
code = baseline_code("cfg5_n16384")
cfg = AdmmConfig(mu=5.0)
ch = Awgn(2.5, 0.5)
decode_synth(code, ch, cfg, seed=1, point=1, trial0=0, batch=256)
torch.cuda.synchronize()
lib = _lib.load()
buf = (ctypes.c_uint64 * 8)()
_lib.check(lib.admm_cluster_phase_profile(1, None))
r = decode_synth(code, ch, cfg, seed=1, point=1, trial0=0, batch=a.frames)
torch.cuda.synchronize()
_lib.check(lib.admm_cluster_phase_profile(0, buf))
names = ["scatter-in", "variable", "x-send", "barrier A", "check", "msg-send", "barrier B+decide"]
it = buf[7]
tot = sum(buf[:7])
print(f"iterations seen by CTA 0: {it}, cycles/iteration {tot / max(it, 1):.0f}")
for k, n in enumerate(names):
    print(f"  {n:18s} {buf[k] / max(it, 1):8.0f} cycles  {100 * buf[k] / max(tot, 1):5.1f} %")
