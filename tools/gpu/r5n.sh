# final verification pass: smoke, GPU suite, bench (default), reference arm, C4/C5 artefacts
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/r5n_pytest.log 2>&1; echo "rc=$?" >> $O/r5n_pytest.log
tail -2 $O/r5n_pytest.log
timeout 600 python bench.py > $O/r5n_bench.json 2> $O/r5n_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 200 --warmup 5 > $O/r5n_bench_ref.json 2> $O/r5n_bench_ref.err; echo "ref rc=$?"
timeout 900 python tools/bench_c4.py --tiles 10000 --steps 5 > $O/r5n_c4.json 2>/dev/null
timeout 900 python tools/bench_c4.py --tiles 10000 --steps 3 --groups intensity,shape,moments,glcm,glrlm,glszm,ngtdm > $O/r5n_c4_all7.json 2>/dev/null
timeout 900 python tools/bench_c5.py --steps 3 > $O/r5n_c5.json 2>/dev/null
timeout 600 python tools/bench_groups.py --steps 20 > $O/r5n_groups.jsonl 2>/dev/null
python - <<'PY'
import json
O = "gpurun_out"
d = json.load(open(f"{O}/r5n_bench.json")); r = json.load(open(f"{O}/r5n_bench_ref.json"))
print("c2", d["value"], d["ms_per_step"], "e2e", d["e2e"]["value"], "raw", d["e2e"]["raw_rows"]["value"], "ref", r["value"], d["clocks"])
c4 = json.load(open(f"{O}/r5n_c4.json")); print("c4", c4["ms_per_step"], "e2e", c4["e2e"]["value"])
a7 = json.load(open(f"{O}/r5n_c4_all7.json")); print("c4all", a7["ms_per_step"], "e2e", a7["e2e"]["value"])
c5 = json.load(open(f"{O}/r5n_c5.json")); print("c5", c5["ms_per_step"])
for l in open(f"{O}/r5n_groups.jsonl"):
    g = json.loads(l); print(g["config"], g["groups"], g["ms_per_step"], round(g["mp_per_s"]))
PY
