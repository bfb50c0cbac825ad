cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/r3u_pytest.log 2>&1; echo "rc=$?" >> $O/r3u_pytest.log
tail -4 $O/r3u_pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 > $O/r3u_bench.json 2> $O/r3u_bench.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('$O/r3u_bench.json'))
print('value', d['value'], 'ms', d['ms_per_step']); print('e2e', json.dumps(d['e2e'])); print('clocks', d.get('clocks'))"
