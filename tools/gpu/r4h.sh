cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/r4h_smoke.log 2>&1; tail -1 $O/r4h_smoke.log
timeout 900 python bench.py > $O/r4h_bench.json 2> $O/r4h_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > $O/r4h_ref.json 2> $O/r4h_ref.err; echo "ref rc=$?"
python -c "
import json
d=json.load(open('$O/r4h_bench.json')); print('ours', d['value'], d['ms_per_step'], 'e2e', d['e2e']['value'], 'steps', d['steps'], d['warmup'], 'roof', d['roofline']['kernel'], d['roofline']['frac'], 'clocks', d['clocks'])
r=json.load(open('$O/r4h_ref.json')); print('ref', r['value'], r.get('cpu_baseline'))"
