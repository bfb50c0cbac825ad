cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/r4q_pytest.log 2>&1; echo "rc=$?" >> $O/r4q_pytest.log
tail -2 $O/r4q_pytest.log
timeout 900 python tools/bench_c4.py --tiles 10000 --steps 3 --groups intensity,shape,moments,glcm,glrlm,glszm,ngtdm > $O/r4q_c4_all7.json 2> /dev/null
python -c "
import json; d=json.load(open('$O/r4q_c4_all7.json'))
print('c4all', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']), {k: round(v,2) for k,v in d['kernels_ms_per_step'].items() if v > 1})"
timeout 900 python tools/bench_c5.py --steps 3 > $O/r4q_c5.json 2>/dev/null
python -c "
import json; d=json.load(open('$O/r4q_c5.json')); print('c5', d['ms_per_step'])"
