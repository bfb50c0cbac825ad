cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/r4n_pytest.log 2>&1; echo "rc=$?" >> $O/r4n_pytest.log
tail -2 $O/r4n_pytest.log
timeout 600 python tools/bench_groups.py --steps 20 > $O/r4n_groups.jsonl 2> /dev/null
python -c "
import json
for l in open('$O/r4n_groups.jsonl'):
    d=json.loads(l); print(d['config']['workload'][:60], round(d['ms_per_step'],3), round(d['value']))"
timeout 600 python tools/bench_c4.py --tiles 10000 --steps 5 > $O/r4n_c4.json 2>/dev/null
python -c "
import json; d=json.load(open('$O/r4n_c4.json')); print('c4', d['ms_per_step'], 'e2e', d['e2e']['value'])"
