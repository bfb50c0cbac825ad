cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests/test_batch.py -m gpu -q -p no:cacheprovider -x > $O/r3q.log 2>&1; echo "rc=$?" >> $O/r3q.log
tail -15 $O/r3q.log
timeout 600 python bench.py --steps 20 --warmup 5 > $O/r3q_bench.json 2> $O/r3q_bench.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('$O/r3q_bench.json'))
print('value', d['value'], 'ms', d['ms_per_step']); print('e2e', json.dumps(d['e2e']))"
tail -3 $O/r3q_bench.err
