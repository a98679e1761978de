"""The pipelined host-to-host API (paper_1204_0556_b200.pipeline), i.e. the
e2e path bench.py measures: results equal decode_batch on the same LLRs."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_host_pipeline_matches_decode_batch(cuda_ok, dtype):
    from paper_1204_0556_b200 import AdmmConfig, baseline_code, decode_batch
    from paper_1204_0556_b200.channels import awgn_gammas_device
    from paper_1204_0556_b200.pipeline import HostPipeline

    code = baseline_code("cfg2_n1008")
    cfg = AdmmConfig(mu=5.0)
    chunks_dev = [awgn_gammas_device(n, code.n_vars, db, code.design_rate, seed=k, dtype=dtype)
                  for k, (n, db) in enumerate([(300, 2.0), (517, 2.5), (64, 3.0)])]
    host = [g.cpu().pin_memory() for g in chunks_dev]
    pipe = HostPipeline(code, cfg, dtype=dtype, max_batch=600)
    out = pipe.run(host)
    torch.cuda.synchronize()
    assert pipe.h2d_bytes_per_run(host) == sum(h.numel() * h.element_size() for h in host)
    for g, r in zip(chunks_dev, out):
        ref = decode_batch(g, code, cfg, dtype=dtype, want_x=False, want_hard=True)
        assert torch.equal(r.iterations, ref.iterations.cpu())
        assert torch.equal(r.flags, ref.flags.cpu())
        assert torch.equal(r.weight, ref.weight.cpu())
        assert torch.equal(r.hard, ref.hard.cpu())
    # the pipeline is reusable and deterministic
    out2 = pipe.run(host)
    torch.cuda.synchronize()
    assert all(torch.equal(a.hard, b.hard) for a, b in zip(out, out2))
    with pytest.raises(ValueError):
        pipe.run([torch.zeros((601, code.n_vars), dtype=dtype).pin_memory()])


def test_host_pipeline_reused_outputs(cuda_ok):
    from paper_1204_0556_b200 import AdmmConfig, baseline_code, decode_batch
    from paper_1204_0556_b200.channels import awgn_gammas_device
    from paper_1204_0556_b200.pipeline import HostPipeline

    code = baseline_code("cfg1_n96")
    g = awgn_gammas_device(200, code.n_vars, 2.0, code.design_rate, seed=4, dtype=torch.float32)
    host = [g[:120].cpu().pin_memory(), g[120:].cpu().pin_memory()]
    pipe = HostPipeline(code, AdmmConfig(mu=5.0), dtype=torch.float32, max_batch=128, reuse_outputs=True)
    a = pipe.run(host)
    torch.cuda.synchronize()
    first = [r.hard.clone() for r in a]
    b = pipe.run(host)
    torch.cuda.synchronize()
    assert all(x.hard.data_ptr() == y.hard.data_ptr() for x, y in zip(a, b))  # buffers reused
    ref = decode_batch(g, code, AdmmConfig(mu=5.0), dtype=torch.float32, want_x=False, want_hard=True)
    assert torch.equal(torch.cat([r.hard for r in b]), ref.hard.cpu())
    assert all(torch.equal(x, y.hard) for x, y in zip(first, b))
