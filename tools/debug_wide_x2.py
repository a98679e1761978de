import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
from paper_1204_0556_b200 import AdmmConfig, Awgn, baseline_code, decode_batch, synth_llr  # noqa: E402
code = baseline_code("cfg5_n16384")
B = 4608
g = synth_llr(code.n_vars, Awgn(2.5, code.design_rate), seed=5, point=0, trial0=0, batch=B, dtype=torch.float32)
cfg = AdmmConfig(mu=5.0, epsilon=1e-300, t_max=1)
w = decode_batch(g, code, cfg, dtype=torch.float32, want_x=True, engine="wide")
torch.cuda.synchronize()
exp = (-(g / 5.0) / 3.0).clamp(0, 1)
for f in (2048, 2049, 2050, 2112):
    bad = ((w.x[f] - exp[f]).abs() > 1e-5).nonzero().flatten()
    print(f, "bad vars", bad.numel(), bad[:20].tolist())
    if bad.numel():
        i = bad[0].item()
        print("   x", w.x[f, i].item(), "exp", exp[f, i].item(), "g", g[f, i].item(),
              "exp from other frames?", [(ff, round(exp[ff, i].item(), 5)) for ff in range(f - 2, f + 3)])
