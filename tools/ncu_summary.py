"""Summarise an ncu report: key SOL metrics, stall reasons, DRAM bytes, top source lines.
usage: python tools/ncu_summary.py report.ncu-rep [--lines N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
nlines = int(sys.argv[sys.argv.index("--lines") + 1]) if "--lines" in sys.argv else 25


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
h, u, v = raw[0], raw[1], raw[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct", "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum", "l1tex__t_sector_hit_rate.pct"]
for a, b, c in zip(h, u, v):
    if a in want:
        print(f"{a:60s} {b:12s} {c}")
print("-- stalls (pc samples)")
st = [(float(c.replace(",", "")), a) for a, b, c in zip(h, u, v)
      if a.startswith("smsp__pcsamp_warps_issue_stalled_") and not a.endswith("not_issued") and c not in ("", "n/a")]
tot = sum(x for x, _ in st) or 1
for x, a in sorted(st, reverse=True)[:10]:
    print(f"  {a.replace('smsp__pcsamp_warps_issue_stalled_', ''):30s} {100 * x / tot:5.1f}%")
rows = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "sass,cuda"))))
cur = hdr = None
out = []
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0] not in ("", "Function Name"):
        d = dict(zip(hdr, r))
        try:
            s = int(d["Warp Stall Sampling (All Samples)"])
        except Exception:
            continue
        out.append((s, cur, r[0], r[1].strip()[:100], d.get("stall_long_sb"), d.get("stall_barrier"), d.get("stall_lg")))
tot = sum(o[0] for o in out) or 1
out.sort(reverse=True)
print("-- top source lines (share of samples; long_sb / barrier / lg)")
for o in out[:nlines]:
    print(f"{100 * o[0] / tot:5.1f}% {o[1]}:{o[2]} {o[3]}  [{o[4]}/{o[5]}/{o[6]}]")
