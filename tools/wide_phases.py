"""Phase breakdown of the wide kernel (admm_wide_phase_profile) on cfg5."""
import ctypes
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1204_0556_b200 import AdmmConfig, Awgn, _lib, baseline_code, decode_synth  # noqa: E402

code = baseline_code("cfg5_n16384")
cfg = AdmmConfig(mu=5.0)
ch = Awgn(2.5, code.design_rate)
B = int(os.environ.get("B", "65536"))
dt = torch.float64 if os.environ.get("DT", "f32") == "f64" else torch.float32
lib = _lib.load()
decode_synth(code, ch, cfg, seed=1, point=1, trial0=0, batch=4096, dtype=dt)
torch.cuda.synchronize()
_lib.check(lib.admm_wide_phase_profile(1, None))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
r = decode_synth(code, ch, cfg, seed=1, point=1, trial0=0, batch=B, dtype=dt)
e1.record()
torch.cuda.synchronize()
out = (ctypes.c_uint64 * 8)()
_lib.check(lib.admm_wide_phase_profile(0, out))
ms = e0.elapsed_time(e1)
eu = int(r.iterations.sum()) * code.n_edges
passes = out[6]
names = ["stepA(V:G0+C:G1)", "sync", "slotsG1+sync", "stepB(C:G0+V:G1)", "sync", "slotsG0+sync"]
tot = sum(out[:6])
print(f"B={B} {ms:.1f} ms  {eu / ms / 1e6:.1f} G eu/s  passes={passes}  us/pass={1e3 * ms / max(passes, 1):.1f}")
print("  ".join(f"{n}={100 * out[k] / tot:.1f}%" for k, n in enumerate(names)))
print("cycles/pass:", "  ".join(f"{n}={out[k] / max(passes, 1):.0f}" for k, n in enumerate(names)))
