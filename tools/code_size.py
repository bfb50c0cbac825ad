"""Static SASS size (and optional ncu per-address metrics) per source phase of process_roi.
usage: code_size.py <cubin> <kernel-substring> [ncu_sass.csv]"""
import collections, csv, re, subprocess, sys
cubin, target = sys.argv[1], sys.argv[2]
PH = [("load1", 216, 270), ("load2", 271, 313), ("sort", 314, 327), ("cmom", 328, 351),
      ("pct+mad+rmad", 352, 395), ("mode_hist", 396, 456), ("edge", 457, 610), ("int_out", 611, 656),
      ("moments", 657, 780), ("glcm", 781, 1000)]
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
    if m and not pending:
        addr_line[int(m.group(1), 16)] = last
        continue
    if m:
        ch = []
        for p in pending:
            ch += [(f.split("/")[-1], int(l)) for f, l in re.findall(r'File "([^"]+)", line (\d+)', p)]
        pending = []
        ins = [c for c in ch if c[0] == "fx_roi.cu" and 200 <= c[1] <= 1000]
        cur = ins[0] if ins else (ch[0] if ch else ("?", 0))
        nm = "other"
        for p, lo, hi in PH:
            if cur[0] == "fx_roi.cu" and lo <= cur[1] <= hi:
                nm = p
        addr_line[int(m.group(1), 16)] = nm
        last = nm
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
print(f"{'phase':14s} {'sass':>6s} {'exec%':>6s} {'stall%':>6s}")
for nm, n in stat.most_common():
    print(f"{nm:14s} {n:6d} {100*ex[nm]/te:6.1f} {100*sm[nm]/ts:6.1f}")
