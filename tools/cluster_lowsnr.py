import sys, torch
sys.path.insert(0, ".")
from paper_1204_0556_b200 import AdmmConfig, Awgn, baseline_code, decode_synth
code = baseline_code("cfg5_n16384")
cfg = AdmmConfig(mu=5.0)
for snr in (1.5, 2.0):
    ch = Awgn(snr, code.design_rate)
    decode_synth(code, ch, cfg, seed=1, point=0, trial0=0, batch=64)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r = decode_synth(code, ch, cfg, seed=1, point=0, trial0=0, batch=2048)
    e1.record(); torch.cuda.synchronize()
    it = int(r.iterations.to(torch.int64).sum())
    ms = e0.elapsed_time(e1)
    print(f"snr {snr}: {ms:.1f} ms, {it*code.n_edges/ms/1e6:.1f} G eu/s, mean iters {it/2048:.1f}, converged {int(r.converged.sum())}, iter checksum {it}")
