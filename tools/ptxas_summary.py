"""Summarise a `-Xptxas -v` log: registers / spills per kernel (demangled)."""
import re, subprocess, sys

def parse(path):
    out = {}
    name = None
    for line in open(path):
        m = re.search(r"Compiling entry function '(\S+)' for", line)
        if m:
            name = m.group(1)
            continue
        m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m and name:
            out.setdefault(name, {})["spill"] = (int(m.group(1)), int(m.group(2)))
        m = re.search(r"Used (\d+) registers", line)
        if m and name:
            out.setdefault(name, {})["regs"] = int(m.group(1))
    return out

def demangle(names):
    r = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True)
    return r.stdout.splitlines()

if __name__ == "__main__":
    logs = [parse(p) for p in sys.argv[1:]]
    names = list(logs[0])
    dem = demangle(names)
    for n, d in zip(names, dem):
        short = re.sub(r"\(.*", "", d).replace("admm::", "").replace("void ", "")
        cols = []
        for lg in logs:
            e = lg.get(n, {})
            cols.append(f"{e.get('regs','-'):>4} {str(e.get('spill','-')):>12}")
        if len(logs) == 1 or len(set(cols)) > 1:
            print(f"{short[:90]:<90} " + " | ".join(cols))
