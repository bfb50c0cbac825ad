cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests/test_batch.py -m gpu -q -p no:cacheprovider -x -k "packed or banded" 2>&1 | tail -3
timeout 600 python bench.py --steps 20 --warmup 5 > $O/r3z_bench.json 2> $O/r3z_bench.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('$O/r3z_bench.json'))
print('value', d['value'], 'ms', d['ms_per_step']); print('e2e', d['e2e']['value'], d['e2e']['h2d_bytes_per_step'], 'raw', d['e2e']['raw_rows'])"
