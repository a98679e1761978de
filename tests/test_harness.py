"""Monte-Carlo harness (paper_1204_0556_b200.simulator): host logic on CPU,
GPU runs against the reference harness's own CSV output (golden)."""
import numpy as np
import pytest
import torch

from conftest import golden_code, load_golden
from paper_1204_0556_b200.simulator import CSV_COLUMNS, DecoderRef, TrialStats, stats_to_csv


def test_csv_formatting_matches_reference_layout():
    s = TrialStats("admm", "bsc", 0.03, 107, 96, 0.5, trials=300, word_errors=8, bit_errors=60,
                   iter_sum_correct=3174, iter_sum_erroneous=7956)
    text = stats_to_csv([s], timing=False)
    head, row = text.splitlines()
    assert head.split(",") == CSV_COLUMNS
    assert row == "admm,bsc,0.03,0.5,96,300,8,60,0.0266667,0.00208333,37.1,10.8699,994.5,,,,0,107"
    empty = stats_to_csv([TrialStats("admm", "bsc", 0.1, 1, 10, 0.5)])
    assert empty.splitlines()[1] == "admm,bsc,0.1,0.5,10,0,0,0,0,0,,,,,,,0,1"


def test_merge_and_validation():
    a = TrialStats("admm", "awgn", 2.0, 1, 10, 0.5, trials=3, word_errors=1, bit_errors=2)
    b = TrialStats("admm", "awgn", 2.0, 1, 10, 0.5, trials=5, word_errors=2, bit_errors=1)
    m = a.merge(b)
    assert (m.trials, m.word_errors, m.bit_errors) == (8, 3, 3)
    with pytest.raises(ValueError):
        a.merge(TrialStats("admm", "bsc", 2.0, 1, 10, 0.5))
    with pytest.raises(ValueError):
        DecoderRef("nope")
    with pytest.raises(NotImplementedError):
        DecoderRef("dual-ascent").admm_config()
    from paper_1204_0556_b200 import BpConfig

    assert DecoderRef("bp").admm_config() == BpConfig()


@pytest.mark.gpu
@pytest.mark.parametrize("batch", [64, 4096])
def test_gpu_sweep_reproduces_reference_csv(cuda_ok, batch):
    """fp64 GPU decode + the reference's frame seeding: byte-identical CSV."""
    from paper_1204_0556_b200 import AdmmConfig, Awgn, Bsc
    from paper_1204_0556_b200.simulator import run_point, sweep

    f = load_golden("harness.npz")
    code = golden_code(f)
    dec = DecoderRef("admm", AdmmConfig(mu=3.0))
    got = stats_to_csv(sweep(code, [Bsc(0.03), Awgn(2.5, code.design_rate)], dec, n_trials=300, seed=107,
                             batch_size=batch), timing=False)
    assert got == str(f["csv_sweep"])
    got_t = stats_to_csv([run_point(code, Bsc(0.05), dec, target_errors=20, max_trials=5000, seed=108,
                                    point_index=2, batch_size=batch)], timing=False)
    assert got_t == str(f["csv_target"])


@pytest.mark.gpu
def test_device_frames_statistically_match(cuda_ok):
    """In-kernel Philox frames vs the reference's numpy frames: WER within
    2 standard errors (tests/test_acceptance.py:242-244 tolerance)."""
    from paper_1204_0556_b200 import AdmmConfig, Awgn, baseline_code
    from paper_1204_0556_b200.simulator import run_point

    code = baseline_code("cfg1_n96")
    dec = DecoderRef("admm", AdmmConfig(mu=5.0))
    ch = Awgn(3.0, code.design_rate)
    a = run_point(code, ch, dec, n_trials=4000, seed=5, frames="reference")
    b = run_point(code, ch, dec, n_trials=20000, seed=5, frames="device", dtype=torch.float32)
    se = np.sqrt(a.wer * (1 - a.wer) / a.trials + b.wer * (1 - b.wer) / b.trials)
    assert abs(a.wer - b.wer) <= 2 * se + 1e-4
    # device frames are a pure function of (seed, point, trial): batch-size invariant
    c = run_point(code, ch, dec, n_trials=20000, seed=5, frames="device", dtype=torch.float32, batch_size=777)
    assert stats_to_csv([b], timing=False) == stats_to_csv([c], timing=False)


@pytest.mark.gpu
def test_device_frames_fast_accounting_equals_full(cuda_ok):
    """The device-frame path counts bit errors from the kernel's weights and
    resolves ML accounting only for certified error words; the per-trial
    records equal a full computation from the hard decisions and LLRs of every
    trial (BSC near the LP threshold, so certified errors occur)."""
    from paper_1204_0556_b200 import AdmmConfig, Bsc, baseline_code, decode_synth, synth_llr
    from paper_1204_0556_b200.simulator import _decode_wave

    code = baseline_code("cfg1_n96")
    cfg = AdmmConfig(mu=5.0)
    ch = Bsc(0.09)
    sent = np.zeros(code.n_vars, dtype=np.uint8)
    we, be, it, _, ml = _decode_wave(code, ch, cfg, sent, 3, 1, range(0, 3000), frames="device",
                                     dtype=torch.float64, device="cuda", engine="auto")
    full = decode_synth(code, ch, cfg, seed=3, point=1, trial0=0, batch=3000, dtype=torch.float64, want_hard=True)
    gam = synth_llr(code.n_vars, ch, seed=3, point=1, trial0=0, batch=3000, dtype=torch.float64)
    hard = full.hard.to(torch.float64)
    be_full = full.hard.to(torch.int64).sum(dim=1)
    ml_full = (be_full > 0) & full.codeword & ((gam * hard).sum(dim=1) < 0)
    assert np.array_equal(be, be_full.cpu().numpy())
    assert np.array_equal(we, (be_full > 0).cpu().numpy())
    assert np.array_equal(it, full.iterations.cpu().numpy().astype(np.int64))
    assert np.array_equal(ml, ml_full.cpu().numpy())
    assert int(ml_full.sum()) > 0 or int(((be_full > 0) & full.codeword).sum()) > 0
