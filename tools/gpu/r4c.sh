cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/r4c_pytest.log 2>&1; echo "rc=$?" >> $O/r4c_pytest.log
tail -3 $O/r4c_pytest.log
for raw in 10 30; do
FXG_PACK_RAW=$raw timeout 600 python tools/bench_c4.py --tiles 2000 --steps 2 --e2e-tiles 2000 > $O/r4c_c4.json 2>/dev/null
python -c "
import json; d=json.load(open('$O/r4c_c4.json'))
print('raw% $raw c4 e2e', d['e2e']['value'])"
done
timeout 900 python tools/bench_c4.py --tiles 10000 --steps 3 --groups intensity,shape,moments,glcm,glrlm,glszm,ngtdm > $O/r4c_c4_all7.json 2> /dev/null
python -c "
import json; d=json.load(open('$O/r4c_c4_all7.json'))
print('c4 all7 ms', d['ms_per_step'], 'e2e', json.dumps(d['e2e']))"
