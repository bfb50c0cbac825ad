cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/r4i_pytest.log 2>&1; echo "rc=$?" >> $O/r4i_pytest.log
tail -3 $O/r4i_pytest.log
for i in 1 2; do
timeout 600 python bench.py --steps 20 --warmup 5 > $O/r4i_bench.json 2>/dev/null
python -c "
import json; d=json.load(open('$O/r4i_bench.json'))
print('value', d['value'], 'e2e', d['e2e']['value'], 'raw', d['e2e']['raw_rows']['value'])"
done
CALLS=5 timeout 300 python tools/pack_trace.py 2>&1 | awk '/call 3:/{f=1} f' | grep "device\|call" | head -16
