"""Debug: wide kernel vs sharded kernel on the same trials (cfg5 code)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1204_0556_b200 import AdmmConfig, Awgn, baseline_code, decode_synth  # noqa: E402

code = baseline_code("cfg5_n16384")
cfg = AdmmConfig(mu=5.0)
ch = Awgn(2.5, code.design_rate)
B = int(os.environ.get("B", "2304"))
dt = torch.float64 if os.environ.get("DT", "f64") == "f64" else torch.float32
ref = torch.cat([decode_synth(code, ch, cfg, seed=1, point=1, trial0=lo, batch=min(256, B - lo), dtype=dt,
                              engine="streaming").iterations for lo in range(0, B, 256)])
w = decode_synth(code, ch, cfg, seed=1, point=1, trial0=0, batch=B, dtype=dt, engine="wide")
torch.cuda.synchronize()
print("kernel", w.info["kernel"], "ref kernel(256)", "mean it", ref.float().mean().item(), w.iterations.float().mean().item())
bad = (w.iterations != ref).nonzero().flatten()
print("mismatches", bad.numel(), "of", B)
print("first", bad[:40].tolist())
print("ref it", ref[bad[:20]].tolist())
print("wide it", w.iterations[bad[:20]].tolist())
