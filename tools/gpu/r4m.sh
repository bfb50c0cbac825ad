cd $GRAFT_REPO_ROOT
O=gpurun_out
: > $O/r4m.log
for v in lib_alt/g12 lib_alt/g14 lib_alt/g16 lib_alt/g20; do
  FX_GROUPS=intensity,moments,glcm FXG_LIB=$v/libfxg.so timeout 300 python tools/kbench.py c2 5 2>&1 | tail -1 | sed "s#^#$v #" | cut -c1-60,110-220 >> $O/r4m.log
  FXG_LIB=$v/libfxg.so timeout 300 python tools/kbench.py c3 10 2>&1 | tail -1 | sed "s#^#$v #" | cut -c1-200 >> $O/r4m.log
  FXG_LIB=$v/libfxg.so timeout 600 python tools/bench_c4.py --tiles 2000 --steps 3 --e2e-tiles 8 > $O/r4m_c4.json 2>/dev/null
  python -c "
import json; d=json.load(open('$O/r4m_c4.json')); k=d['kernels_ms_per_step']
print('$v c4', round(d['ms_per_step'],2), 'S0', round(k.get('k_roi_s0',0),2), 'S1', round(k.get('k_roi_s1',0),2), 'S2', round(k.get('k_roi_s2',0),2))" >> $O/r4m.log
done
cat $O/r4m.log
