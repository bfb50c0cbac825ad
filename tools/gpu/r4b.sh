cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests/test_batch.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -2
FXG_PACK_TRACE=1 timeout 600 python tools/bench_c4.py --tiles 2000 --steps 2 --e2e-tiles 2000 > $O/r4b_c4.json 2> $O/r4b_c4.err; echo "c4 rc=$?"
grep batch-pack $O/r4b_c4.err | tail -8
python -c "
import json; d=json.load(open('$O/r4b_c4.json'))
print('c4 ms', d['ms_per_step'], 'e2e', json.dumps(d['e2e']))"
timeout 600 python tools/bench_c4.py --tiles 10000 --steps 5 > $O/r4b_c4full.json 2>/dev/null
python -c "
import json; d=json.load(open('$O/r4b_c4full.json'))
print('c4 full ms', d['ms_per_step'], 'e2e', json.dumps(d['e2e']))"
