"""bench.py's reference arm (the CPU oracle, no GPU needed) prints the one
JSON line the driver parses, with the keys the contract requires."""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--workload", "cfg1",
                          "--steps", "1", "--warmup", "0", "--cpu-frames", "8"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference"
    assert d["value"] > 0 and d["unit"] == "frames/s" and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert "workload" in d["config"]


def _stub(gpus, *extra):
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--stub", "--gpus", str(gpus), "--frames", "1000",
                          *extra], capture_output=True, text=True, timeout=600, cwd=ROOT,
                         env={k: v for k, v in __import__("os").environ.items()
                              if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")})
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_gpus_flag_relaunches_ranks_and_merges_counters():
    """`bench.py --gpus 2` without a launcher re-launches itself with two
    ranks (torch.distributed.run); the rank logic (shards, counter
    all-reduce, max-over-ranks) is rehearsed over gloo with a stub decoder:
    the merged counters equal the single-rank run (strong scaling of cfg5)."""
    one, two = _stub(1), _stub(2)
    assert one["n_gpus"] == 1 and two["n_gpus"] == 2
    assert one["counters"] == two["counters"] and two["frames"] == 2000
    three = _stub(3, "--workload", "cfg5")
    assert three["n_gpus"] == 3 and three["counters"] == one["counters"]
