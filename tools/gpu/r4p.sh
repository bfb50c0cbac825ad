cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python tools/bench_c4.py --tiles 10000 --steps 3 --groups intensity,shape,moments,glcm,glrlm,glszm,ngtdm > $O/r4p_c4_all7.json 2> /dev/null
python -c "
import json; d=json.load(open('$O/r4p_c4_all7.json'))
print('c4 all7 ms', d['ms_per_step'], 'e2e', d['e2e']['value'], 'raw', d['e2e']['raw_rows']['value'])
print({k: round(v,2) for k,v in d['kernels_ms_per_step'].items()})"
timeout 900 python tools/bench_c5.py --steps 3 > $O/r4p_c5.json 2>/dev/null
python -c "
import json; d=json.load(open('$O/r4p_c5.json')); print('c5', d['ms_per_step'], d['kernels_ms_per_step_rank0'].get('k_roi_b'))"
