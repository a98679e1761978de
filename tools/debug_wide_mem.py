"""Debug: wide kernel vs sharded kernel on device LLRs (decode_batch), direct and retiring paths."""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1204_0556_b200 import AdmmConfig, Awgn, baseline_code, decode_batch, synth_llr  # noqa: E402

code = baseline_code("cfg5_n16384")
cfg = AdmmConfig(mu=5.0)
B = int(os.environ.get("B", "4608"))
dt = torch.float64 if os.environ.get("DT", "f32") == "f64" else torch.float32
g = synth_llr(code.n_vars, Awgn(2.5, code.design_rate), seed=5, point=0, trial0=0, batch=B, dtype=dt)
ref = torch.cat([decode_batch(g[lo:lo + 256], code, cfg, dtype=dt, want_x=False, engine="streaming").iterations
                 for lo in range(0, B, 256)])
torch.cuda.synchronize()
for want_x in (False, True):
    t0 = time.time()
    w = decode_batch(g, code, cfg, dtype=dt, want_x=want_x, engine="wide")
    torch.cuda.synchronize()
    bad = (w.iterations != ref).nonzero().flatten()
    print("want_x", want_x, "kernel", w.info["kernel"], f"{time.time() - t0:.2f}s", "mean it", ref.float().mean().item(),
          w.iterations.float().mean().item(), "mismatches", bad.numel(), bad[:10].tolist())
