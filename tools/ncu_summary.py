"""Summarise an ncu --page raw --csv dump into profiles/<name>.md + traffic json.
usage: ncu_summary.py raw.csv out.md traffic.json "title" """
import csv, json, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr, units = rows[0], rows[1]
keys = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'smsp__inst_executed.sum', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'lts__t_sector_hit_rate.pct',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed']
scale = {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9}
lines = [f"# {sys.argv[4]}", ""]
traffic = {}
for r in rows[2:]:
    name = r[hdr.index('Kernel Name')].split('(')[0].replace('void ', '').split('::')[-1]
    lines.append(f"## {name}")
    tb = 0.0
    for k in keys:
        if k in hdr:
            i = hdr.index(k)
            lines.append(f"- {k}: {r[i]} {units[i]}")
            if k.startswith('dram__bytes_'):
                tb += float(r[i].replace(',', '')) * scale.get(units[i], 1)
    lines.append(f"- dram traffic per launch (read+write): {tb / 1e6:.1f} MB")
    lines.append("")
    traffic[name] = int(tb)
open(sys.argv[2], 'w').write("\n".join(lines))
json.dump({"source": sys.argv[2] + " (ncu --set full; dram__bytes_read.sum + dram__bytes_write.sum)",
           "bytes_per_launch": traffic}, open(sys.argv[3], 'w'), indent=1)
print("\n".join(lines))
