cd $GRAFT_REPO_ROOT
O=gpurun_out
for v in paper_2603_12016_b200/lib lib_alt/tm3 lib_alt/tm2; do
  FXG_LIB=$v/libfxg.so timeout 600 python tools/bench_c4.py --tiles 2000 --steps 3 --e2e-tiles 8 --groups intensity,shape,moments,glcm,glrlm,glszm,ngtdm > $O/r4t.json 2>/dev/null
  python -c "
import json; d=json.load(open('$O/r4t.json')); k=d['kernels_ms_per_step']
print('$v', round(d['ms_per_step'],2), 'k_roi_t', round(k.get('k_roi_t',0),2))"
done
