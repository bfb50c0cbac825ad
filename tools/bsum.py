import json, sys
for line in sys.stdin:
    line = line.strip()
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    print("value", d.get("value"), d.get("unit"), "ms/step", d.get("ms_per_step"), "e2e", d.get("e2e", {}).get("value"))
    print("kernels", d.get("kernels_ms_per_step"))
    print("roofline", d.get("roofline"))
    print("cpu", d.get("cpu_baseline"), "clocks", d.get("clocks"), "launches", d.get("gpu_launches"))
