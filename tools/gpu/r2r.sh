cd $GRAFT_REPO_ROOT
O=gpurun_out
for v in "" lib_alt/s0w48 lib_alt/s0w56 lib_alt/s0n1024 lib_alt/s0w48n1024; do
  L=${v:+$v/libfxg.so}
  echo "== ${v:-default}"
  FXG_LIB=$L timeout 120 python tools/kbench.py c2 20 2>&1 | tail -1
  FXG_LIB=$L timeout 300 python tools/bench_c4.py --tiles 4000 --steps 3 --e2e-tiles 16 2>/dev/null | python -c "import sys,json; d=json.load(sys.stdin); print('c4', round(d['ms_per_step'],2), {k:round(v,2) for k,v in d['kernels_ms_per_step'].items()})"
  FXG_LIB=$L timeout 300 python tools/bench_c4.py --tiles 4000 --steps 2 --e2e-tiles 16 --groups intensity,shape,moments,glcm,glrlm,glszm,ngtdm 2>/dev/null | python -c "import sys,json; d=json.load(sys.stdin); print('c4all', round(d['ms_per_step'],2), {k:round(v,2) for k,v in d['kernels_ms_per_step'].items()})"
done > $O/r2r_s0var.log 2>&1
for v in lib_alt/s0w48 lib_alt/s0w48n1024; do
  FXG_LIB=$v/libfxg.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_scale_parity.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -1 | sed "s|^|$v |"
done >> $O/r2r_s0var.log 2>&1
cat $O/r2r_s0var.log
