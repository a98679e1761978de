"""Monte-Carlo harness throughput on device frames (run_point)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1204_0556_b200 import AdmmConfig, Awgn, baseline_code  # noqa: E402
from paper_1204_0556_b200.simulator import DecoderRef, run_point  # noqa: E402

for name, snr, n in (("cfg2_n1008", 2.0, 262144), ("cfg5_n16384", 2.5, 65536)):
    code = baseline_code(name)
    dec = DecoderRef("admm", AdmmConfig(mu=5.0))
    ch = Awgn(snr, code.design_rate)
    run_point(code, ch, dec, n_trials=4096, seed=1, frames="device", dtype=torch.float32, batch_size=4096)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st = run_point(code, ch, dec, n_trials=n, seed=1, frames="device", dtype=torch.float32, batch_size=65536)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"{name} {snr} dB: {n / dt:,.0f} frames/s through run_point (wer {st.wer:.3g}, {n} trials)")
