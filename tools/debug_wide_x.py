"""Debug: x after t_max iterations, wide (memory LLRs) vs sharded."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1204_0556_b200 import AdmmConfig, Awgn, baseline_code, decode_batch, synth_llr  # noqa: E402

code = baseline_code("cfg5_n16384")
B = 4608
g = synth_llr(code.n_vars, Awgn(2.5, code.design_rate), seed=5, point=0, trial0=0, batch=B, dtype=torch.float32)
for T in (1, 2, 3):
    cfg = AdmmConfig(mu=5.0, epsilon=1e-300, t_max=T)
    w = decode_batch(g, code, cfg, dtype=torch.float32, want_x=True, engine="wide")
    r = torch.cat([decode_batch(g[lo:lo + 256], code, cfg, dtype=torch.float32, want_x=True, engine="streaming").x
                   for lo in range(0, B, 256)])
    torch.cuda.synchronize()
    d = (w.x - r).abs().max(dim=1).values
    bad = (d > 1e-4).nonzero().flatten()
    print("T", T, "iters", w.iterations[:4].tolist(), "bad frames", bad.numel(), bad[:12].tolist(),
          "maxdiff f0", d[0].item(), "f2", d[2].item())
    if T == 1:
        x0 = (-(g[:4] / 5.0) / 3.0).clamp(0, 1)
        print("  expected-x diff f0..3", (w.x[:4] - x0).abs().max(dim=1).values.tolist())
