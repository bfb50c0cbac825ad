"""Attribute ncu per-instruction counts to CUDA source lines, across a kernel and
its noinline callees (ncu lists them back to back; each function's start is found
by matching its opcode sequence from nvdisasm).

usage: sass_attr.py <ncu_sass.csv> <cubin> <kernel-substring> [top]
env:   SRCF=fx_roi_s.cu  OUTER=lo:hi  (attribute inlined code to the outermost frame
       of SRCF whose line lies in [lo, hi], e.g. the body of process_s)
       PHASES=name:lo:hi,...  (per-phase totals over the attributed line)
"""
import collections
import csv
import os
import re
import subprocess
import sys

csvf, cubin, target = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
SRCF = os.environ.get("SRCF", "fx_roi_s.cu")
OUT = [int(v) for v in os.environ.get("OUTER", "0:0").split(":")]
PH = [(p.split(":")[0], int(p.split(":")[1]), int(p.split(":")[2]))
      for p in os.environ.get("PHASES", "").split(",") if p]

dis = subprocess.run(["nvdisasm", "-gi", "-c", cubin], capture_output=True, text=True).stdout
funcs, cur, chain = {}, None, None
for line in dis.splitlines():
    m = re.match(r"^\s*\.text\.(\S+):", line) or re.match(r"^(_Z\S+):$", line)
    if m:
        cur = m.group(1)
        funcs.setdefault(cur, [])
        continue
    if "//## File" in line:
        chain = [(f.split("/")[-1], int(l)) for f, l in re.findall(r'"([^"]+)", line (\d+)', line)]
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m and cur:
        op = re.sub(r"^\{?\s*(@!?U?P\w+\s+)?", "", m.group(2)).split()[0] if m.group(2).strip() else "?"
        funcs[cur].append((int(m.group(1), 16), op, chain))

rows = list(csv.reader(open(csvf)))
hdr = rows[1]
ia, isrc = hdr.index("Address"), hdr.index("Source")
ie, isamp = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
lst = []
for r in rows[2:]:
    try:
        a = int(r[ia], 16)
    except (ValueError, IndexError):
        continue
    txt = r[isrc].strip()
    op = re.sub(r"^\{?\s*(@!?U?P\w+\s+)?", "", txt).split()[0] if txt else "?"
    lst.append((a, op, float(r[ie] or 0), float(r[isamp] or 0)))
ops = [x[1] for x in lst]


def locate(seq):
    n = min(24, len(seq))
    pat = [s[1] for s in seq[:n]]
    for i in range(len(ops) - n + 1):
        if ops[i:i + n] == pat:
            return i
    return None


def attr_line(chain):
    if not chain:
        return ("?", 0)
    if OUT[1]:
        inside = [c for c in chain if c[0] == SRCF and OUT[0] <= c[1] <= OUT[1]]
        if inside:
            return inside[-1]
    mine = [c for c in chain if c[0] == SRCF]
    return mine[0] if mine else chain[0]


agg = collections.defaultdict(lambda: [0.0, 0.0])
covered = 0
for name, seq in funcs.items():
    if not seq:
        continue
    if target not in name and not any(target in n and name.split("$")[-1] in n for n in funcs):
        continue
    i = locate(seq)
    if i is None:
        continue
    for k, (_, op, ch) in enumerate(seq):
        if i + k >= len(lst):
            break
        e, s = lst[i + k][2], lst[i + k][3]
        agg[attr_line(ch)][0] += e
        agg[attr_line(ch)][1] += s
        covered += 1
tot_e = sum(x[2] for x in lst)
tot_s = sum(x[3] for x in lst)
got_e = sum(v[0] for v in agg.values())
print(f"ncu rows {len(lst)}  attributed rows {covered}  inst {got_e:.4g} of {tot_e:.4g}")
if PH:
    ph = collections.defaultdict(lambda: [0.0, 0.0])
    for (f, l), (e, s) in agg.items():
        nm = "other"
        for n, lo, hi in PH:
            if f == SRCF and lo <= l <= hi:
                nm = n
        ph[nm][0] += e
        ph[nm][1] += s
    for nm, (e, s) in sorted(ph.items(), key=lambda kv: -kv[1][0]):
        print(f"PHASE {nm:14s} inst {100 * e / tot_e:5.1f}%  stall {100 * s / max(tot_s, 1):5.1f}%")
for k, (e, s) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{k[0]}:{k[1]:5d}  inst {100 * e / tot_e:5.1f}%  stall {100 * s / max(tot_s, 1):5.1f}%")
