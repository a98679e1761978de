"""Benchmark: BASELINE config 2 sweep through the sm_100a ADMM-LP decoder.

One STEP = decoding the BASELINE.json config-2 workload once: the (3,6)
n=1008 girth-6 code, all-zero codeword over BPSK/AWGN at Eb/N0 = 1.5, 1.75,
..., 3.0 dB (7 points), 65536 frames per point, mu=5, eps=1e-5, T_max=1000,
rho=1.9 (the reference default).  Inputs are seeded synthetic LLRs generated
on the device before timing (1.85 GB fp32 per step -- far larger than the
126 MB L2, so no L2 flush is needed between steps).

``value`` = decoded frames/s of the whole job (all ranks), device-timed with
CUDA events, inputs resident in HBM.  ``e2e`` = the same metric through the
public pipelined host API (paper_1204_0556_b200.pipeline): pinned host LLRs
in, host hard decisions / iterations / flags out, copies inside the timed
region.  ``--impl reference`` times the CPU oracle (numpy restatement of the
reference, oracle/admm_oracle.py) on the box's host cores on a bounded sample
of the same workload.

Multi-GPU (torchrun): every rank decodes its own frames (weak scaling; trial
indices are sharded by rank), and one NCCL all-reduce of int64 counters
merges the statistics.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

POINTS_DB = [1.5, 1.75, 2.0, 2.25, 2.5, 2.75, 3.0]
FRAMES_PER_POINT = 65536
MU, EPS, TMAX, RHO = 5.0, 1e-5, 1000, 1.9
METRIC = "decoded frames/s (ADMM-LP, config 2 sweep)"
BYTES_PER_EDGE_UPDATE = {"f32": 28, "f64": 56}  # 6s + 3s/d_v, d_v = 3


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--dtype", choices=["f32", "f64"], default="f32")
    ap.add_argument("--frames", type=int, default=FRAMES_PER_POINT, help="frames per SNR point per GPU")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample")
    ap.add_argument("--cpu-frames", type=int, default=0, help="oracle frames per point (0 = auto)")
    ap.add_argument("--workload", choices=["cfg2", "cfg5"], default="cfg2",
                    help="cfg2: headline sweep (default); cfg5: n=16384 large-block case, 1M frames/point "
                         "sharded over the ranks (strong scaling), fused on-GPU frame synthesis")
    ap.add_argument("--chunk", type=int, default=65536, help="cfg5: frames per decode call")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


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
        rows = []
        for line in self.path.read_text().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
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
# CPU leg (oracle) -- used for cpu_baseline and --impl reference
# ---------------------------------------------------------------------------
def cpu_sample(code, frames_per_point: int, workers: int, seed_base: int = 0):
    """Decode a bounded, SNR-stratified sample of the workload with the CPU
    oracle over `workers` processes.  Returns (seconds, frames, edge_updates)."""
    from oracle import admm_oracle as O

    g = O.Graph.of(code)
    rate = 1.0 - code.n_checks / code.n_vars
    gam = np.concatenate([
        np.array([O.trial_gamma_awgn(code.n_vars, db, rate, 1, k, seed_base + t) for t in range(frames_per_point)])
        for k, db in enumerate(POINTS_DB)])
    t0 = time.perf_counter()
    iters, conv, hard = O.decode_parallel(gam, g, O.Params(mu=MU, epsilon=EPS, t_max=TMAX, rho=RHO), workers)
    dt = time.perf_counter() - t0
    return dt, len(gam), int(iters.sum()) * code.n_edges


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def run_reference(args):
    """--impl reference: the CPU oracle on the host cores, same metric."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from paper_1204_0556_b200.codes import baseline_code

    code = baseline_code("cfg2_n1008")
    workers = os.cpu_count() or 1
    fpp = args.cpu_frames or 16 * workers
    times, frames, eus = [], 0, 0
    for s in range(args.warmup + args.steps):
        dt, nf, eu = cpu_sample(code, fpp, workers, seed_base=s * fpp)
        if s >= args.warmup:
            times.append(dt)
            frames += nf
            eus += eu
    total = sum(times)
    val = frames / total
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "frames/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded AWGN LLRs, all-zero codeword)",
        "config": {"workload": "cfg2 sweep (n=1008 (3,6) girth-6, 1.5-3.0 dB step 0.25, mu=5, eps=1e-5, "
                               "T_max=1000, rho=1.9)", "sample_frames_per_point": fpp},
        "edge_updates_per_s": eus / total,
        "cpu_baseline": {"value": val, "unit": "frames/s", "cores": workers, "kind": "port",
                         "sample": f"{fpp} frames per SNR point x 7 points per step, oracle/admm_oracle.py "
                                   f"(numpy restatement of polylp.decode), {workers} processes, {cpu_model()}"},
        "e2e": {"value": val, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU leg
# ---------------------------------------------------------------------------
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1204_0556_b200 import AdmmConfig, baseline_code, decode_batch
    from paper_1204_0556_b200.channels import Awgn, awgn_gammas_device
    from paper_1204_0556_b200.pipeline import HostPipeline

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    code = baseline_code("cfg2_n1008")
    cfg = AdmmConfig(mu=MU, epsilon=EPS, t_max=TMAX, rho=RHO)
    tdt = torch.float32 if args.dtype == "f32" else torch.float64
    F = args.frames
    # Seeded device-side LLRs; rank r owns trial block r (weak scaling).
    gam = [awgn_gammas_device(F, code.n_vars, db, code.design_rate, seed=1000003 * (k + 1) + 7919 * rank,
                              device=dev, dtype=tdt) for k, db in enumerate(POINTS_DB)]
    stream = torch.cuda.current_stream(dev)

    def step(collect=False):
        outs = []
        for k in range(len(POINTS_DB)):
            r = decode_batch(gam[k], code, cfg, dtype=tdt, want_x=True, validate=False, stream=stream)
            outs.append(r)
        return outs

    # warm-up (also builds the device graph) and the deterministic work count
    outs = None
    for _ in range(max(args.warmup, 1)):
        outs = step()
    torch.cuda.synchronize(dev)
    iters_sum = sum(int(o.iterations.sum()) for o in outs)
    edge_updates = iters_sum * code.n_edges
    info = outs[0].info

    # timed region: K steps, per-launch events for the roofline
    clocks = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clocks.start()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps * len(POINTS_DB))]
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    n = 0
    for s in range(args.steps):
        for k in range(len(POINTS_DB)):
            ev[n][0].record(stream)
            decode_batch(gam[k], code, cfg, dtype=tdt, want_x=True, validate=False, stream=stream)
            ev[n][1].record(stream)
            n += 1
    t1.record(stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    elapsed = t0.elapsed_time(t1) / 1e3
    launch_s = sum(a.elapsed_time(b) for a, b in ev) / 1e3 / n
    if world > 1:
        t = torch.tensor([elapsed], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = float(t.item())

    # statistics of one step, merged with ONE all-reduce of int64 counters
    from paper_1204_0556_b200.distributed import allreduce_counters, counters_as_dict, counters_from_results

    cnt = torch.zeros(8, dtype=torch.int64, device=dev)
    for k in range(len(POINTS_DB)):
        o = decode_batch(gam[k], code, cfg, dtype=tdt, want_x=False, want_hard=True, validate=False)
        cost = (gam[k].to(torch.float64) * o.hard.to(torch.float64)).sum(dim=1)
        cnt += counters_from_results(o.iterations, o.weight, o.converged, o.codeword, cost, code.n_edges)
    cnt = counters_as_dict(allreduce_counters(cnt))

    frames_per_step = F * len(POINTS_DB)
    value = world * frames_per_step * args.steps / elapsed
    eu_total = world * edge_updates * args.steps / elapsed

    # roofline of the dominant kernel (the resident decode kernel is the only one)
    peak_path = ROOT / "MEASURED_PEAKS.json"
    peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
    if peak_path.exists():
        peak, peak_src = float(json.loads(peak_path.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    bpe = BYTES_PER_EDGE_UPDATE[args.dtype]
    per_launch_bytes = bpe * edge_updates / len(POINTS_DB)
    achieved = per_launch_bytes / launch_s / 1e9
    traffic = None
    tpath = ROOT / "profiles" / "traffic.json"
    if tpath.exists():
        try:
            bpf = json.loads(tpath.read_text()).get(f"bytes_per_frame_{args.dtype}")
            traffic = None if bpf is None else bpf * F  # ncu DRAM bytes per frame x frames per launch
        except Exception:
            traffic = None

    # e2e through the pipelined host API
    e2e = None
    if not args.no_e2e:
        pipe = HostPipeline(code, cfg, dtype=tdt, device=dev, max_batch=F)
        host = [g.cpu().pin_memory() for g in gam]
        pipe.run(host[:2])  # warm
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for s in range(args.steps):
            res = pipe.run(host)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        e_el = e0.elapsed_time(e1) / 1e3
        if world > 1:
            t = torch.tensor([e_el], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_el = float(t.item())
        e2e = {"value": world * frames_per_step * args.steps / e_el, "unit": "frames/s",
               "h2d_bytes_per_step": pipe.h2d_bytes_per_run(host),
               "d2h_bytes_per_step": pipe.d2h_bytes_per_run(host)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        workers = os.cpu_count() or 1
        fpp = args.cpu_frames or 16 * workers
        dt, nf, eu = cpu_sample(code, fpp, workers)
        cpu = {"value": nf / dt, "unit": "frames/s", "cores": workers, "kind": "port",
               "edge_updates_per_s": eu / dt,
               "sample": f"{fpp} frames per SNR point x 7 points (SNR-stratified sample of the same workload), "
                         f"oracle/admm_oracle.py over {workers} processes, {cpu_model()}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * elapsed / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": args.dtype,
            "data": "synthetic (seeded device AWGN LLRs, all-zero codeword)",
            "config": {"workload": "cfg2 sweep: (3,6) n=1008 girth-6 code, AWGN 1.5-3.0 dB step 0.25, "
                                   f"{F} frames/point/GPU, mu=5, eps=1e-5, T_max=1000, rho=1.9",
                       "frames_per_step_per_gpu": frames_per_step, "parallelism": f"frame-shard x{world}",
                       "l2": "inputs 1.85 GB/step >> 126 MB L2 (no flush needed)",
                       "engine": info},
            "edge_updates_per_s": eu_total,
            "mean_iterations": iters_sum / frames_per_step,
            "stats_one_step_all_ranks": cnt,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "bytes_model": f"{bpe} B per edge-update (two-kernel HBM schedule, SURVEY 8d) x "
                                        f"{edge_updates // len(POINTS_DB)} edge-updates per launch",
                         "kernel": f"resident engine {info.get('engine')} (1 generic, 2 regular)",
                         "avg_launch_ms": launch_s * 1e3,
                         "note": "fused on-chip design: the HBM-model bytes are never moved (edge state stays in "
                                 "registers/SMEM); `traffic` is the ncu DRAM bytes per launch; the real bound is SM "
                                 "instruction issue (DESIGN.md 3.4)"},
            "gpu_launches": args.steps * len(POINTS_DB),
            "clocks": clk,
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_cfg5(args):
    """BASELINE config 5: (3,6) n=16384 girth-6 code, BSC p=0.04 and AWGN 2.5 dB,
    1,048,576 frames per point sharded over the ranks (strong scaling).  LLRs
    are synthesised inside the decode kernel from (seed, point, trial), so
    the statistics are identical for every GPU count."""
    import torch
    import torch.distributed as dist

    from paper_1204_0556_b200 import AdmmConfig, Awgn, Bsc, baseline_code, decode_synth
    from paper_1204_0556_b200.distributed import allreduce_counters, counters_as_dict, counters_from_results, shard

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    code = baseline_code("cfg5_n16384")
    cfg = AdmmConfig(mu=MU, epsilon=EPS, t_max=TMAX, rho=RHO)
    tdt = torch.float32 if args.dtype == "f32" else torch.float64
    total = args.frames if args.frames != FRAMES_PER_POINT else 1048576
    points = [Bsc(0.04), Awgn(2.5, code.design_rate)]
    mine = shard(total, rank, world)
    stream = torch.cuda.current_stream(dev)

    def step(collect=False):
        outs = []
        for k, ch in enumerate(points):
            for lo in range(mine.start, mine.stop, args.chunk):
                n = min(args.chunk, mine.stop - lo)
                r = decode_synth(code, ch, cfg, seed=1, point=k, trial0=lo, batch=n, dtype=tdt, stream=stream)
                if collect:
                    outs.append(r)
        return outs

    outs = step(collect=True)
    for _ in range(max(args.warmup - 1, 0)):
        step()
    torch.cuda.synchronize(dev)
    iters_sum = sum(int(o.iterations.to(torch.int64).sum()) for o in outs)
    edge_updates = iters_sum * code.n_edges
    cnt = torch.zeros(8, dtype=torch.int64, device=dev)
    for o in outs:
        cnt += counters_from_results(o.iterations, o.weight, o.converged, o.codeword,
                                     torch.zeros(o.iterations.numel(), device=dev), code.n_edges)
    cnt = counters_as_dict(allreduce_counters(cnt))
    info = outs[0].info
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
    elapsed = t0.elapsed_time(t1) / 1e3
    n_launch = len(outs)
    launch_s = elapsed / args.steps / n_launch
    if world > 1:
        t = torch.tensor([elapsed], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = float(t.item())
        e = torch.tensor([edge_updates], dtype=torch.int64, device=dev)
        dist.all_reduce(e)
        edge_updates_all = int(e.item())
    else:
        edge_updates_all = edge_updates
    peak = float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]) \
        if (ROOT / "MEASURED_PEAKS.json").exists() else 6650.0
    bpe = BYTES_PER_EDGE_UPDATE[args.dtype]
    achieved = bpe * edge_updates / n_launch / launch_s / 1e9
    if rank == 0:
        line = {
            "metric": "decoded frames/s (ADMM-LP, config 5 large block)", "value": len(points) * total * args.steps / elapsed,
            "unit": "frames/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * elapsed / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": args.dtype, "data": "synthetic (in-kernel Philox LLRs keyed by seed/point/trial)",
            "config": {"workload": f"cfg5: (3,6) n=16384 girth-6, BSC 0.04 + AWGN 2.5 dB, {total} frames/point total",
                       "parallelism": f"frame-shard x{world}", "chunk": args.chunk, "engine": info},
            "edge_updates_per_s": edge_updates_all * args.steps / elapsed,
            "mean_iterations": iters_sum / (len(points) * len(mine)),
            "stats_one_step_all_ranks": cnt,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": None, "bytes_model": f"{bpe} B per edge-update (SURVEY 8d)",
                         "kernel": "streaming_decode_kernel", "avg_launch_ms": launch_s * 1e3},
            "gpu_launches": args.steps * n_launch,
            "clocks": clk, "e2e": None, "cpu_baseline": None,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.workload == "cfg5" and args.impl == "ours":
        run_cfg5(args)
        return
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
