"""Opcode histogram of one kernel's SASS (cuobjdump -sass of an object file).
   python tools/sass_hist.py build/resident_f32.o 'resident_regular_kernelIfLi6ELi3ELi2ELi4ELi4E' [more objects...]
Counts the instructions between the first and the last backward branch target
(the hot loops) as well as the whole kernel."""
import collections, re, subprocess, sys

def kernels(obj):
    txt = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    cur, out = None, {}
    for line in txt.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            out[cur] = []
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m and cur:
            out[cur].append((int(m.group(1), 16), m.group(2)))
    return out

def hist(ins):
    h = collections.Counter()
    for _, s in ins:
        s = re.sub(r"^@!?U?P\d+\s+", "", s)
        op = s.split()[0].split(".")[0]
        h[op] += 1
    return h

if __name__ == "__main__":
    pat = sys.argv[2]
    hs = []
    for obj in [sys.argv[1]] + sys.argv[3:]:
        ks = kernels(obj)
        name = [k for k in ks if pat in k]
        assert name, (obj, pat)
        ins = ks[name[0]]
        # loop region: from the smallest backward-branch target to the last backward branch
        lo, hi = None, None
        for a, s in ins:
            m = re.search(r"BRA\S*\s+.*?0x([0-9a-f]+)", s)
            if m and int(m.group(1), 16) < a:
                t = int(m.group(1), 16)
                lo = t if lo is None else min(lo, t)
                hi = a
        loop = [(a, s) for a, s in ins if lo is not None and lo <= a <= hi]
        hs.append((name[0], hist(ins), hist(loop), len(ins), len(loop)))
    ops = sorted(set().union(*[h[2] for h in hs]), key=lambda o: -hs[0][2][o])
    print("kernel:", hs[0][0])
    print(f"{'op':<12}" + "".join(f"{'loop' + str(i):>8}" for i in range(len(hs))))
    for o in ops:
        print(f"{o:<12}" + "".join(f"{h[2][o]:>8}" for h in hs))
    print(f"{'TOTAL loop':<12}" + "".join(f"{h[4]:>8}" for h in hs))
    print(f"{'TOTAL all':<12}" + "".join(f"{h[3]:>8}" for h in hs))


def loops(ins):
    """(target, branch address) of every backward branch."""
    out = []
    for a, s in ins:
        m = re.search(r"BRA\S*\s+.*?0x([0-9a-f]+)", s)
        if m and int(m.group(1), 16) < a:
            out.append((int(m.group(1), 16), a))
    return out
