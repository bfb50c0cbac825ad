cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/r5a_pytest.log 2>&1; echo "rc=$?" >> $O/r5a_pytest.log
tail -2 $O/r5a_pytest.log
timeout 600 python bench.py > $O/r5a_bench.json 2>/dev/null
python -c "
import json; d=json.load(open('$O/r5a_bench.json')); print('value', d['value'], d['ms_per_step'], 'e2e', d['e2e']['value'], 'gpu_launches', d['gpu_launches'], 'spot', d.get('parity_spot_check'))"
