cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests/test_batch.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -1
for i in 1 2; do
timeout 600 python bench.py --steps 20 --warmup 5 > $O/r5k_bench.json 2>/dev/null
python -c "
import json; d=json.load(open('$O/r5k_bench.json')); print('e2e', d['e2e']['value'], d['e2e']['h2d_bytes_per_step'], 'raw', d['e2e']['raw_rows']['value'])"
done
timeout 600 python tools/bench_c4.py --tiles 2000 --steps 3 --e2e-tiles 2000 > $O/r5k_c4.json 2>/dev/null
python -c "
import json; d=json.load(open('$O/r5k_c4.json')); print('c4 e2e', d['e2e']['value'], 'raw', d['e2e']['raw_rows']['value'])"
