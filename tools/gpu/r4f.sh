cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python tools/bench_c4.py --tiles 10000 --steps 3 --groups intensity,shape,moments,glcm,glrlm,glszm,ngtdm > $O/r4f_c4_all7.json 2> $O/r4f.err
python -c "
import json; d=json.load(open('$O/r4f_c4_all7.json'))
print('c4 all7 ms', d['ms_per_step'], 'e2e', d['e2e']['value'], 'raw', d['e2e']['raw_rows']['value'], d['e2e']['matches_device_table'])
print(d['kernels_ms_per_step'])"
timeout 900 python -m pytest tests/test_batch.py tests/test_gpu_parity.py tests/test_random_parity.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -2
