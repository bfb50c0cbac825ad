"""Per-phase executed-instruction mix (opcode histogram) from ncu SASS csv.
usage: phase_mix.py cubin kernel csv phase1,phase2  (PHASES env as code_size.py)"""
import collections, csv, os, re, subprocess, sys
cubin, target, csvf, want = sys.argv[1], sys.argv[2], sys.argv[3], sys.argv[4].split(",")
SRCF = os.environ.get("SRCF", "fx_roi_s.cu")
PH = [tuple([p.split(":")[0]] + [int(v) for v in p.split(":")[1:]]) for p in os.environ["PHASES"].split(",")]
LO = min(p[1] for p in PH); HI = max(p[2] for p in PH)
dis = subprocess.run(["nvdisasm", "-gi", "-c", cubin], capture_output=True, text=True).stdout
infn, pending, amap, last = False, [], {}, "other"
for line in dis.splitlines():
    if line.startswith(".text.") or re.match(r"^_Z\S+:$", line):
        infn = target in line; continue
    if not infn: continue
    if "//## File" in line: pending.append(line); continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", line)
    if not m: continue
    if pending:
        ch = []
        for p in pending: ch += [(f.split("/")[-1], int(l)) for f, l in re.findall(r'File "([^"]+)", line (\d+)', p)]
        pending = []
        ins = [c for c in ch if c[0] == SRCF and LO <= c[1] <= HI]
        cur = ins[0] if ins else ("?", 0)
        last = "other"
        for n, lo, hi in PH:
            if cur[0] == SRCF and lo <= cur[1] <= hi: last = n
    amap[int(m.group(1), 16)] = last
rows = list(csv.reader(open(csvf))); hdr = rows[1]
ia, isrc, ie = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed")
base = None; mix = collections.defaultdict(collections.Counter); nroi = float(os.environ.get("NROI", "50000"))
for r in rows[2:]:
    try: a = int(r[ia], 16)
    except ValueError: continue
    base = a if base is None else base
    src = r[isrc].strip(); o = src.split()[1] if src.startswith("@") else src.split()[0]
    mix[amap.get(a - base, "?")][o.split(".")[0]] += float(r[ie] or 0)
for ph in want:
    tot = sum(mix[ph].values())
    print(ph, f"{tot / nroi:.0f}/ROI:", ", ".join(f"{o} {e / nroi:.0f}" for o, e in mix[ph].most_common(16)))
