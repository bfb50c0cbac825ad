"""Join an ncu SASS source page (csv) with nvdisasm line info: per-source-line
instruction counts and stall samples.  usage: sass_lines.py <ncu.csv> <cubin> <func>"""
import csv, re, subprocess, sys, collections
csvf, cubin, func = sys.argv[1:4]
import os
PHASE_FILE = os.environ.get("PHASE_FILE", "")
PHASE_LO, PHASE_HI = int(os.environ.get("PHASE_LO", "0")), int(os.environ.get("PHASE_HI", "1000000"))
PHASES = [tuple(p.split(":")) for p in os.environ.get("PHASES", "").split(",") if p]
if True:
    dis = subprocess.run(["nvdisasm", "-gi", "-c", cubin], capture_output=True, text=True).stdout
    i = dis.find(f"{func}:")
    dis = dis[i:]
    j = dis.find("//---------------------", 10)
    dis = dis[:j] if j > 0 else dis
cur = None
addr2 = {}
chain, fresh = [], True
for line in dis.splitlines():
    if "//## File" in line:
        # nvdisasm prints one marker line per inline level, innermost first
        if fresh:
            chain, fresh = [], False
        chain += [(f.split("/")[-1], int(l)) for f, l in re.findall(r'"([^"]+)", line (\d+)', line)[:1]]
        cur = chain[0]
        if PHASE_FILE:
            inside = [c for c in chain if c[0] == PHASE_FILE and PHASE_LO <= c[1] <= PHASE_HI]
            if inside:
                cur = inside[0]
        continue
    m = re.match(r'\s+/\*([0-9a-f]{4,})\*/', line)
    if m and cur:
        addr2[int(m.group(1), 16)] = cur
        fresh = True
rows = list(csv.reader(open(csvf)))
hdr = rows[1]
ia, ie, isamp = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
agg = collections.defaultdict(lambda: [0, 0])
base = None
tot = [0, 0]
for r in rows[2:]:
    try:
        a = int(r[ia], 16)
        base = a if base is None else base
        a -= base
        e = float(r[ie] or 0); s = float(r[isamp] or 0)
    except ValueError:
        continue
    k = addr2.get(a, ("?", 0))
    agg[k][0] += e; agg[k][1] += s
    tot[0] += e; tot[1] += s
print(f"total inst {tot[0]:.3g} samples {tot[1]:.0f}")
if PHASES:
    ph = collections.defaultdict(lambda: [0, 0])
    for (f, l), (e, s_) in agg.items():
        name = "other"
        for nm, lo, hi in PHASES:
            if f == PHASE_FILE and int(lo) <= l <= int(hi):
                name = nm
        ph[name][0] += e; ph[name][1] += s_
    for nm, (e, s_) in sorted(ph.items(), key=lambda kv: -kv[1][1]):
        print(f"PHASE {nm:12s} inst {100*e/tot[0]:5.1f}%  stall {100*s_/tot[1]:5.1f}%")
for k, (e, s) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:int(sys.argv[4]) if len(sys.argv) > 4 else 40]:
    print(f"{k[0]}:{k[1]:5d}  inst {100*e/tot[0]:5.1f}%  stall {100*s/tot[1]:5.1f}%")
