"""Benchmark of the sm_100a ADMM-LP decoder on the BASELINE.json workloads.

Default (what the driver runs): BASELINE config 5, the metric's
"1/2/4/8 B200" case -- the (3,6) n=16384 girth-6 code, all-zero codeword,
BSC p=0.04 and BPSK/AWGN 2.5 dB, 1,048,576 frames per point SHARDED over
the GPUs (strong scaling), mu=5, eps=1e-5, T_max=1000, rho=1.9 (the
reference default), fp32.  One STEP = decoding both points once (2,097,152
frames over all GPUs).

``value`` = decoded frames/s of the whole job, device-timed with CUDA events
(max over ranks).  The frames' LLRs are synthesised inside the decode kernel
from (seed, point, trial) (Philox; csrc/synth.cuh), so no input is read at
all.  ``e2e`` = the same metric through the public host API
(paper_1204_0556_b200.pipeline.HostPipeline): pinned host fp32 LLR blocks
copied in, per-frame iterations / flags / weights copied out, H2D,
decode and D2H overlapped on three streams; the host LLRs are a pool of
distinct frames per point (synth_llr of the point's first trials, staged
once before timing) that the blocks cycle through -- every step copies
all 2 x 1M frames' LLRs (h2d_bytes_per_step).  ``cpu_baseline`` and
``--impl reference`` time the CPU oracle (numpy restatement of the reference,
oracle/admm_oracle.py) on the box's host cores on a bounded sample.

``--workload cfg1..cfg4`` run the other BASELINE configs (weak scaling: every
rank decodes its own frames, device-resident LLRs).

Multi-GPU: ``--gpus N`` without a launcher re-launches itself under
torch.distributed.run with N ranks (NCCL); under torchrun the world size
must equal --gpus.  Frames are independent: rank r decodes its shard, and
one NCCL all-reduce of int64 counters merges the statistics.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from dataclasses import dataclass
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

MU, EPS, TMAX, RHO = 5.0, 1e-5, 1000, 1.9
BYTES_PER_EDGE_UPDATE = {"f32": 28, "f64": 56}  # 6s + 3s/d_v, d_v = 3


@dataclass(frozen=True)
class Workload:
    name: str
    code: str          # paper_1204_0556_b200.codes.BASELINE_CODES key
    points: tuple      # ("awgn", snr_db) or ("bsc", p)
    frames: int        # frames per point (per GPU for weak scaling, total for strong)
    scaling: str
    source: str        # "memory" (device LLR arrays) or "synth" (in-kernel Philox)
    text: str


WORKLOADS = {
    "cfg1": Workload("cfg1", "cfg1_n96", (("awgn", 3.0),), 1000, "weak", "memory",
                     "cfg1: (3,6) n=96, AWGN 3.0 dB, 1000 frames"),
    "cfg2": Workload("cfg2", "cfg2_n1008", tuple(("awgn", 1.5 + 0.25 * k) for k in range(7)), 65536, "weak",
                     "memory", "cfg2 sweep: (3,6) n=1008 girth-6, AWGN 1.5-3.0 dB step 0.25, 65536 frames/point"),
    "cfg3": Workload("cfg3", "cfg3_n2640", (("awgn", 2.0), ("awgn", 2.5), ("awgn", 3.0)), 262144, "weak", "memory",
                     "cfg3: (3,6) n=2640 girth-6, AWGN 2.0/2.5/3.0 dB, 262144 frames/point"),
    "cfg4": Workload("cfg4", "cfg4_n1040", tuple(("awgn", 3.5 + 0.5 * k) for k in range(4)), 262144, "weak",
                     "memory", "cfg4: (3,13) n=1040 girth-6, AWGN 3.5-5.0 dB step 0.5, 262144 frames/point"),
    "cfg5": Workload("cfg5", "cfg5_n16384", (("bsc", 0.04), ("awgn", 2.5)), 1048576, "strong", "synth",
                     "cfg5: (3,6) n=16384 girth-6, BSC 0.04 + AWGN 2.5 dB, 1048576 frames/point total"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="cfg5")
    ap.add_argument("--dtype", choices=["f32", "f64"], default="f32")
    ap.add_argument("--frames", type=int, default=0, help="frames per point (0 = the workload's)")
    ap.add_argument("--chunk", type=int, default=262144, help="frames per decode call (synth workloads)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-block", type=int, default=65536, help="frames per host block of the e2e pipeline")
    ap.add_argument("--e2e-pool", type=int, default=131072,
                    help="distinct host LLR frames per point of the e2e leg of synthesised workloads")
    ap.add_argument("--e2e-seconds", type=float, default=60.0,
                    help="time budget of the e2e leg: it times min(--steps, what fits) steps, at least 2")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample")
    ap.add_argument("--cpu-frames", type=int, default=0, help="oracle frames per point (0 = auto)")
    ap.add_argument("--stub", action="store_true",
                    help="CPU rehearsal of the launcher and rank logic: gloo, a stub decoder, no GPU (tests)")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def channel_of(pt, code):
    from paper_1204_0556_b200 import Awgn, Bsc

    kind, val = pt
    return Bsc(val) if kind == "bsc" else Awgn(val, code.design_rate)


# ---------------------------------------------------------------------------
# clocks sampling (B200_PROFILING.md "clocks DURING the timed region")
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = Path(os.environ.get("TMPDIR", "/tmp")) / f"bench_clocks_{os.getpid()}.csv"

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = [[p.strip() for p in line.split(",")] for line in self.path.read_text().splitlines()]
        rows = [r for r in rows if len(r) >= 9]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        load = [s for s in sm if s > 0.5 * (max(mx) if mx else 1)] or sm
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------------------
# CPU leg (oracle) -- cpu_baseline and --impl reference
# ---------------------------------------------------------------------------
def cpu_sample(wl: Workload, code, frames_per_point: int, workers: int, seed_base: int = 0):
    """Decode a bounded, SNR-stratified sample of the workload with the CPU
    oracle over `workers` processes.  Returns (seconds, frames, edge_updates)."""
    from oracle import admm_oracle as O

    g = O.Graph.of(code)
    rate = 1.0 - code.n_checks / code.n_vars
    gam = []
    for k, (kind, val) in enumerate(wl.points):
        for t in range(frames_per_point):
            if kind == "bsc":
                gam.append(O.trial_gamma_bsc(code.n_vars, val, 1, k, seed_base + t))
            else:
                gam.append(O.trial_gamma_awgn(code.n_vars, val, rate, 1, k, seed_base + t))
    gam = np.array(gam)
    t0 = time.perf_counter()
    iters, _conv, _hard = O.decode_parallel(gam, g, O.Params(mu=MU, epsilon=EPS, t_max=TMAX, rho=RHO), workers)
    dt = time.perf_counter() - t0
    # the sample's own statistics, for a cross-check of the GPU line's (same
    # channel points, all-zero codeword: a word error is any non-zero decision)
    cpu_sample.last_stats = {"mean_iterations": float(np.mean(iters)),
                             "word_errors": int(np.count_nonzero(np.asarray(_hard).reshape(len(gam), -1).any(axis=1))),
                             "frames": len(gam)}
    return dt, len(gam), int(iters.sum()) * code.n_edges


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def auto_cpu_frames(wl: Workload, code, workers: int) -> int:
    """About 10-20 s of oracle work: scales with cores, inversely with block length."""
    return max(4, int(16 * workers * 1008 / code.n_vars * 7 / len(wl.points)))


def run_reference(args, wl: Workload):
    """--impl reference: the CPU oracle on the host cores, same metric."""
    rank, _world, _ = dist_env()
    if rank != 0:
        return
    from paper_1204_0556_b200.codes import baseline_code

    code = baseline_code(wl.code)
    workers = os.cpu_count() or 1
    fpp = args.cpu_frames or auto_cpu_frames(wl, code, workers)
    times, frames, eus = [], 0, 0
    for s in range(args.warmup + args.steps):
        dt, nf, eu = cpu_sample(wl, code, fpp, workers, seed_base=s * fpp)
        if s >= args.warmup:
            times.append(dt)
            frames += nf
            eus += eu
    total = sum(times)
    val = frames / total
    line = {
        "impl": "reference", "metric": metric_name(wl), "value": val, "unit": "frames/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": wl.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded AWGN/BSC LLRs, all-zero codeword)",
        "config": {"workload": wl.text + " (mu=5, eps=1e-5, T_max=1000, rho=1.9)", "sample_frames_per_point": fpp},
        "edge_updates_per_s": eus / total,
        "cpu_baseline": {"value": val, "unit": "frames/s", "cores": workers, "kind": "port",
                         "sample": f"{fpp} frames per channel point x {len(wl.points)} points per step, "
                                   f"oracle/admm_oracle.py (numpy restatement of polylp.decode), {workers} processes, "
                                   f"{cpu_model()}"},
        "e2e": {"value": val, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def metric_name(wl: Workload) -> str:
    return {
        "cfg1": "decoded frames/s (ADMM-LP, config 1: n=96, AWGN 3.0 dB)",
        "cfg2": "decoded frames/s (ADMM-LP, config 2 sweep: n=1008, AWGN 1.5-3.0 dB)",
        "cfg3": "decoded frames/s (ADMM-LP, config 3: n=2640, AWGN 2.0/2.5/3.0 dB)",
        "cfg4": "decoded frames/s (ADMM-LP, config 4: (3,13) n=1040, AWGN 3.5-5.0 dB)",
        "cfg5": "decoded frames/s (ADMM-LP, config 5: n=16384, BSC 0.04 + AWGN 2.5 dB, 1M frames/point)",
    }[wl.name]


KERNEL_NAMES = {1: "resident_decode_kernel", 2: "resident_regular_kernel", 3: "sharded_decode_kernel",
                4: "cluster_decode_kernel", 5: "wide_decode_kernel"}


def load_peaks():
    peak_path = ROOT / "MEASURED_PEAKS.json"
    if peak_path.exists():
        d = json.loads(peak_path.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)", float(d.get("sm_max_mhz", 1965.0))
    return 7700.0, "fallback (B200_PROFILING.md nominal HBM3e)", 1965.0


def roofline(args, wl, kernel_id: int, edge_updates_per_launch: float, launch_s: float, sm_mhz, num_sms: int):
    """Roofline of the dominant kernel, per launch.

    * HBM-streaming kernels (wide): ALGORITHMIC bytes = 28 B (fp32) / 56 B
      (fp64) per edge-update (6s + 3s/d_v) x edge-updates per
      launch / launch time, against the measured copy bandwidth.
    * On-chip kernels (resident, cluster): the edge state never touches
      HBM, so the binding resource is instruction issue: warp-instructions
      per launch (ncu inst_executed per edge-update of the same launch shape,
      profiles/traffic.json, x edge-updates per launch) / launch time,
      against 4 issue slots x SMs x the SM clock under load.
    ``traffic`` = ncu dram__bytes_read.sum + dram__bytes_write.sum per launch
    (profiles/traffic.json, same launch shape), null when not captured."""
    hbm_peak, hbm_src, max_mhz = load_peaks()
    name = KERNEL_NAMES.get(kernel_id, "?")
    tr = {}
    tpath = ROOT / "profiles" / "traffic.json"
    key = f"{wl.name}_{args.dtype}_{name}"
    if tpath.exists():
        tr = json.loads(tpath.read_text()).get("launch_shapes", {}).get(key, {})
    traffic = None
    if tr.get("dram_bytes_per_edge_update") is not None:
        traffic = tr["dram_bytes_per_edge_update"] * edge_updates_per_launch
    if kernel_id == 5:
        bpe = BYTES_PER_EDGE_UPDATE[args.dtype]
        achieved = bpe * edge_updates_per_launch / launch_s / 1e9
        return {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s", "frac": achieved / hbm_peak,
                "traffic": traffic, "peak_source": hbm_src, "kernel": name, "avg_launch_ms": launch_s * 1e3,
                "bytes_model": f"{bpe} B per edge-update (SURVEY 8d: 6s + 3s/d_v) x {edge_updates_per_launch:.4g} "
                               f"edge-updates per launch", "traffic_source": tr.get("source")}
    clk = float(sm_mhz or max_mhz)
    peak = 4.0 * num_sms * clk * 1e6 / 1e9  # G warp-instructions/s
    wipe = tr.get("warp_inst_per_edge_update")
    achieved = None if wipe is None else wipe * edge_updates_per_launch / launch_s / 1e9
    return {"bound": "issue", "achieved": achieved, "peak": peak, "unit": "G warp-inst/s",
            "frac": None if achieved is None else achieved / peak, "traffic": traffic,
            "peak_source": f"4 issue slots x {num_sms} SMs x {clk:.0f} MHz (SM clock under load)",
            "kernel": name, "avg_launch_ms": launch_s * 1e3,
            "inst_model": None if wipe is None else f"{wipe:.4g} warp-instructions per edge-update (ncu "
                                                    f"inst_executed, same launch shape) x {edge_updates_per_launch:.4g}",
            "hbm_model_frac": BYTES_PER_EDGE_UPDATE[args.dtype] * edge_updates_per_launch / launch_s / 1e9 / hbm_peak,
            "traffic_source": tr.get("source"),
            "note": "on-chip engine: the HBM model's bytes are never moved (hbm_model_frac > 1 is expected)"}


# ---------------------------------------------------------------------------
# GPU leg
# ---------------------------------------------------------------------------
def run_ours(args, wl: Workload):
    import torch
    import torch.distributed as dist

    from paper_1204_0556_b200 import AdmmConfig, baseline_code, decode_batch, decode_synth, synth_llr
    from paper_1204_0556_b200.channels import awgn_gammas_device, bsc_gammas_device
    from paper_1204_0556_b200.distributed import (allreduce_counters, counters_as_dict, counters_from_results,
                                                  max_over_ranks, shard)
    from paper_1204_0556_b200.pipeline import HostPipeline

    rank, world, local = dist_env()
    if "WORLD_SIZE" in os.environ and world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but the launcher started {world} ranks")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    code = baseline_code(wl.code)
    cfg = AdmmConfig(mu=MU, epsilon=EPS, t_max=TMAX, rho=RHO)
    tdt = torch.float32 if args.dtype == "f32" else torch.float64
    F = args.frames or wl.frames
    stream = torch.cuda.current_stream(dev)
    chans = [channel_of(pt, code) for pt in wl.points]
    gam = None

    if wl.source == "memory":
        # Seeded device-side LLRs; rank r owns its own trial block (weak scaling).
        gam = []
        for k, pt in enumerate(wl.points):
            seed = 1000003 * (k + 1) + 7919 * rank
            if pt[0] == "bsc":
                gam.append(bsc_gammas_device(F, code.n_vars, pt[1], seed=seed, device=dev, dtype=tdt))
            else:
                gam.append(awgn_gammas_device(F, code.n_vars, pt[1], code.design_rate, seed=seed, device=dev,
                                              dtype=tdt))
        frames_local = F * len(wl.points)
        mine = None

        def step(collect=False):
            return [decode_batch(g, code, cfg, dtype=tdt, want_x=False, want_hard=collect, validate=False,
                                 stream=stream) for g in gam]
    else:
        mine = shard(F, rank, world) if wl.scaling == "strong" else range(rank * F, (rank + 1) * F)
        frames_local = len(mine) * len(wl.points)

        def step(collect=False):
            outs = []
            for k, ch in enumerate(chans):
                for lo in range(mine.start, mine.stop, args.chunk):
                    n = min(args.chunk, mine.stop - lo)
                    outs.append(decode_synth(code, ch, cfg, seed=1, point=k, trial0=lo, batch=n, dtype=tdt,
                                             want_hard=collect, stream=stream))
            return outs

    # warm-up (also builds the device graph), the deterministic work count and statistics
    outs = step(collect=True)
    for _ in range(max(args.warmup - 1, 0)):
        step()
    torch.cuda.synchronize(dev)
    iters_sum = sum(int(o.iterations.to(torch.int64).sum()) for o in outs)
    edge_updates = iters_sum * code.n_edges
    n_launch = len(outs)
    cnt = torch.zeros(8, dtype=torch.int64, device=dev)
    for k, o in enumerate(outs):
        if gam is not None:
            cost = (gam[k].to(torch.float64) * o.hard.to(torch.float64)).sum(dim=1)
        else:  # synthesised frames: ML accounting would need the LLRs back; not part of the timed path
            cost = torch.zeros(o.iterations.numel(), dtype=torch.float64, device=dev)
        cnt += counters_from_results(o.iterations, o.weight, o.converged, o.codeword, cost, code.n_edges)
    cnt = counters_as_dict(allreduce_counters(cnt))
    info = outs[0].info
    del outs

    # timed region: K steps
    clocks = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clocks.start()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(args.steps):
        step()
    t1.record(stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    elapsed_local = t0.elapsed_time(t1) / 1e3
    launch_s = elapsed_local / args.steps / n_launch
    elapsed = max_over_ranks(elapsed_local, device=dev)
    totals = torch.tensor([frames_local, edge_updates], dtype=torch.int64, device=dev)
    if world > 1:
        dist.all_reduce(totals)
    frames_all, eu_all = int(totals[0]), int(totals[1])
    value = frames_all * args.steps / elapsed
    kernel_id = info.get("kernel", info.get("engine"))
    roof = roofline(args, wl, kernel_id, edge_updates / n_launch, launch_s, clk.get("sm_mhz"), info["num_sms"])

    # e2e through the pipelined host API: pinned host LLRs in, per-frame
    # results (iterations, flags, weights) out
    e2e = None
    if not args.no_e2e:
        # (multi-GPU: smaller blocks and pool per rank -- the ranks of one node
        # share the host's pinned memory; every step still copies the LLRs of all
        # of the rank's frames)
        blk = min(args.e2e_block, max(frames_local // len(wl.points) // (4 if world > 1 else 1), 1))
        # outputs as in the device-timed leg: per-frame iterations, flags and
        # Hamming weight (the harness's TrialStats inputs; hard decisions on request)
        pipe = HostPipeline(code, cfg, dtype=tdt, device=dev, max_batch=blk, want_hard=False, reuse_outputs=True)
        if gam is not None:
            host = [h for g in gam for h in g.cpu().pin_memory().split(blk)]
            pool_note = "device-generated LLRs of the timed workload, staged in pinned host memory"
        else:
            # a pool of distinct frames per point (the point's first trials of this
            # rank's shard), staged once in pinned host memory; the blocks of a
            # step cycle through it so that every step copies the LLRs of all of
            # the rank's frames
            P = max(blk, min(args.e2e_pool // world, len(mine)) // blk * blk)
            host = []
            for k, ch in enumerate(chans):
                pool = torch.empty((P, code.n_vars), dtype=tdt, pin_memory=True)
                for lo in range(0, P, blk):
                    pool[lo:lo + blk].copy_(synth_llr(code.n_vars, ch, seed=1, point=k, trial0=mine.start + lo,
                                                      batch=blk, dtype=tdt, device=dev))
                blocks = list(pool.split(blk))
                n_blk = -(-len(mine) // blk)
                for j in range(n_blk):
                    b = blocks[j % len(blocks)]
                    rest = len(mine) - j * blk
                    host.append(b if rest >= blk else b[:rest])
            pool_note = (f"host pool of {P} distinct frames per point ({P * code.n_vars * (4 if args.dtype == 'f32' else 8) / 2**30:.1f} "
                         f"GiB pinned), blocks of {blk} frames cycled to cover the rank's {len(mine)} frames per point")
        pipe.run(host)  # warm-up: allocates the pinned result buffers reused by the timed runs
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        # the e2e leg times min(K, what fits --e2e-seconds) steps (same on every
        # rank: `elapsed` is the max over ranks), so a large --steps does not
        # double the run; the count is reported beside the value
        e_steps = max(2, min(args.steps, int(args.e2e_seconds / max(elapsed / args.steps, 1e-9))))
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(e_steps):
            pipe.run(host)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        e_el = max_over_ranks(e0.elapsed_time(e1) / 1e3, device=dev)
        nb = torch.tensor([pipe.h2d_bytes_per_run(host), pipe.d2h_bytes_per_run(host)], dtype=torch.int64, device=dev)
        if world > 1:
            dist.all_reduce(nb)
        e2e = {"value": frames_all * e_steps / e_el, "unit": "frames/s", "steps": e_steps,
               "h2d_bytes_per_step": int(nb[0]), "d2h_bytes_per_step": int(nb[1]),
               "api": "paper_1204_0556_b200.pipeline.HostPipeline.run (decode_batch on three streams)",
               "inputs": pool_note, "block_frames": blk}
        del pipe, host

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        workers = os.cpu_count() or 1
        fpp = args.cpu_frames or auto_cpu_frames(wl, code, workers)
        dt, nf, eu = cpu_sample(wl, code, fpp, workers)
        cpu = {"value": nf / dt, "unit": "frames/s", "cores": workers, "kind": "port", "edge_updates_per_s": eu / dt,
               "sample_stats": getattr(cpu_sample, "last_stats", None),
               "sample": f"{fpp} frames per channel point x {len(wl.points)} points (the same workload's channel "
                         f"points, numpy-seeded trials), oracle/admm_oracle.py over {workers} processes, {cpu_model()}"}

    if rank == 0:
        line = {
            "metric": metric_name(wl), "value": value, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * elapsed / args.steps, "higher_is_better": True,
            "scaling": wl.scaling, "vs_baseline": None, "dtype": args.dtype,
            "data": "synthetic (seeded device LLRs, all-zero codeword)" if gam is not None
            else "synthetic (in-kernel Philox LLRs keyed by seed/point/trial, all-zero codeword)",
            "config": {"workload": wl.text + f" ({F} frames/point{'/GPU' if wl.scaling == 'weak' else ' over all GPUs'}; "
                                             "mu=5, eps=1e-5, T_max=1000, rho=1.9)",
                       "frames_per_step_per_gpu": frames_local, "parallelism": f"frame-shard x{world}",
                       "l2": "inputs >> 126 MB L2 per step (no flush needed)" if gam is not None
                       else "no LLR input (synthesised in the decode kernel); decoder state >> 126 MB L2",
                       "engine": info},
            "edge_updates_per_s": eu_all * args.steps / elapsed,
            "mean_iterations": iters_sum / frames_local,
            "stats_one_step_all_ranks": cnt,
            "roofline": roof,
            "gpu_launches": args.steps * n_launch,
            "clocks": clk,
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_stub(args, wl: Workload):
    """The multi-rank logic of run_ours without a GPU: same sharding,
    counter all-reduce and max-over-ranks timing, over gloo, with a stub
    decoder whose per-trial results are a pure function of the trial index
    (so the merged counters must not depend on the rank count)."""
    import torch
    import torch.distributed as dist

    from paper_1204_0556_b200.distributed import (allreduce_counters, counters_as_dict, counters_from_results,
                                                  max_over_ranks, shard)

    rank, world, _ = dist_env()
    if "WORLD_SIZE" in os.environ and world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but the launcher started {world} ranks")
    if world > 1:
        dist.init_process_group("gloo")
    F = args.frames or wl.frames
    mine = shard(F, rank, world) if wl.scaling == "strong" else range(rank * F, (rank + 1) * F)
    t0 = time.perf_counter()
    cnt = torch.zeros(8, dtype=torch.int64)
    for k in range(len(wl.points)):
        t = torch.arange(mine.start, mine.stop, dtype=torch.int64)
        it = (t * 7 + k) % 23 + 1
        w = torch.where(t % 5 == k, t % 4, torch.zeros_like(t))
        conv = it < 20
        cnt += counters_from_results(it, w, conv, conv, torch.zeros(len(t), dtype=torch.float64), 49152)
    cnt = counters_as_dict(allreduce_counters(cnt))
    elapsed = max_over_ranks(time.perf_counter() - t0)
    if rank == 0:
        print(json.dumps({"stub": True, "n_gpus": world, "frames": cnt["trials"], "counters": cnt,
                          "elapsed_max_s": elapsed, "scaling": wl.scaling}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def relaunch(args) -> int:
    """`--gpus N` without a launcher: re-run this script under
    torch.distributed.run with N ranks on this node (one per GPU)."""
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    wl = WORKLOADS[args.workload]
    if args.gpus < 1:
        raise SystemExit("--gpus must be >= 1")
    if args.impl == "ours" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        raise SystemExit(relaunch(args))
    if args.impl == "reference":
        run_reference(args, wl)
    elif args.stub:
        run_stub(args, wl)
    else:
        run_ours(args, wl)


if __name__ == "__main__":
    main()
