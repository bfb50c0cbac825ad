cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests/test_batch.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -3
timeout 600 python tools/bench_c4.py --tiles 10000 --steps 5 > $O/r4a_c4.json 2> $O/r4a_c4.err; echo "c4 rc=$?"
python -c "
import json; d=json.load(open('$O/r4a_c4.json'))
print('c4 ms', d['ms_per_step'], 'e2e', json.dumps(d['e2e']))"
tail -2 $O/r4a_c4.err
