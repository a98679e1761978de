"""Instructions executed per CUDA source line of one ncu report, normalised
per `--per` units (e.g. CTA-iterations): where the instruction budget goes.
    python tools/ncu_lines.py report.ncu-rep --per N [--top K]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
per = float(sys.argv[sys.argv.index("--per") + 1]) if "--per" in sys.argv else 1.0
top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
cur = hdr = None
out = []
for r in csv.reader(io.StringIO(txt)):
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0] not in ("", "Function Name"):
        d = dict(zip(hdr, r))
        try:
            e = int(d.get("Instructions Executed", "0").replace(",", ""))
        except ValueError:
            continue
        if e:
            out.append((e, cur, r[0], r[1].strip()[:90]))
out.sort(reverse=True)
tot = sum(o[0] for o in out)
print(f"total {tot / per:.0f} warp-instructions per unit")
for e, f, line, src in out[:top]:
    print(f"{e / per:8.0f} {100 * e / tot:5.1f}% {f}:{line} {src}")
