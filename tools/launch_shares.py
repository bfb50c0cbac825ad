"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list into a
markdown table of per-kernel launch counts, total time and share.
usage: launch_shares.py launches.csv out.md "title" """
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if r]
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
ik, iv, iu, im = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit"), \
    hdr.index("Metric Name")
tot = collections.defaultdict(float)
cnt = collections.Counter()
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
for r in rows[hdr_i + 1:]:
    if len(r) <= max(ik, iv, iu, im) or r[im] != "gpu__time_duration.sum":
        continue
    name = r[ik].split("(")[0].replace("void ", "").split("::")[-1]
    tot[name] += float(r[iv].replace(",", "")) * scale.get(r[iu], 1.0)
    cnt[name] += 1
s = sum(tot.values())
out = [f"# {sys.argv[3]}", "", "Cold-cache, serialised launches: compare shares, not absolutes.", "",
       "| kernel | launches | total µs | share |", "|---|---|---|---|"]
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    out.append(f"| {k} | {cnt[k]} | {v:.1f} | {100 * v / s:.1f} % |")
open(sys.argv[2], "w").write("\n".join(out) + "\n")
print("\n".join(out))
