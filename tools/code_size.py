"""Static SASS size and (optionally) ncu per-address executed instructions / stall
samples per source phase.  usage: code_size.py <cubin> <kernel-substring> [ncu_sass.csv]
env: SRCF (source file name), PHASES "name:lo:hi,..." (line ranges)."""
import collections, csv, os, re, subprocess, sys
cubin, target = sys.argv[1], sys.argv[2]
SRCF = os.environ.get("SRCF", "fx_roi_s.cu")
PH = [tuple([p.split(":")[0]] + [int(v) for v in p.split(":")[1:]])
      for p in os.environ.get("PHASES", "mbar:470:501,rowoff+xy:502:533,gather:534:575,sort:576:590,"
                              "pct+medad:591:609,statloop:610:680,flood:681:711,euler:712:754,"
                              "edge_stats:755:839,int_out:840:884,moments:885:999,glcm:1000:1010,"
                              "slowedge:151:250,radix:251:255,kth:256:259,log2:260:266,glcmfn:267:452").split(",")]
LO = min(p[1] for p in PH); HI = max(p[2] for p in PH)
dis = subprocess.run(["nvdisasm", "-gi", "-c", cubin], capture_output=True, text=True).stdout
infn, pending, addr_line, last = False, [], {}, "other"
for line in dis.splitlines():
    if line.startswith(".text.") or re.match(r"^_Z\S+:$", line):
        infn = target in line
        continue
    if not infn:
        continue
    if "//## File" in line:
        pending.append(line)
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", line)
    if not m:
        continue
    if pending:
        ch = []
        for p in pending:
            ch += [(f.split("/")[-1], int(l)) for f, l in re.findall(r'File "([^"]+)", line (\d+)', p)]
        pending = []
        ins = [c for c in ch if c[0] == SRCF and LO <= c[1] <= HI]
        cur = ins[0] if ins else (ch[0] if ch else ("?", 0))
        last = "other"
        for p, lo, hi in PH:
            if cur[0] == SRCF and lo <= cur[1] <= hi:
                last = p
    addr_line[int(m.group(1), 16)] = last
stat = collections.Counter(addr_line.values())
ex, sm = collections.Counter(), collections.Counter()
if len(sys.argv) > 3:
    rows = list(csv.reader(open(sys.argv[3])))
    hdr = rows[1]
    ia, ie, isamp = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    base = None
    for r in rows[2:]:
        try:
            a = int(r[ia], 16)
        except ValueError:
            continue
        base = a if base is None else base
        nm = addr_line.get(a - base, "?")
        ex[nm] += float(r[ie] or 0)
        sm[nm] += float(r[isamp] or 0)
te, ts = max(1, sum(ex.values())), max(1, sum(sm.values()))
print(f"{'phase':14s} {'sass':>6s} {'exec%':>6s} {'stall%':>6s}   (total exec {te:.3g})")
for nm, n in sorted(stat.items(), key=lambda kv: -ex[kv[0]]):
    print(f"{nm:14s} {n:6d} {100*ex[nm]/te:6.1f} {100*sm[nm]/ts:6.1f}")
