cd $GRAFT_REPO_ROOT
O=gpurun_out
for v in "" lib_alt/mask lib_alt/mask_glcm4; do
  L=${v:+$v/libfxg.so}
  echo "== ${v:-default}"
  FXG_LIB=$L timeout 120 python tools/kbench.py c2 40 2>&1 | tail -1
  FXG_LIB=$L timeout 300 python tools/bench_c4.py --tiles 4000 --steps 3 --e2e-tiles 16 2>/dev/null | python -c "import sys,json; d=json.load(sys.stdin); print('c4', round(d['ms_per_step'],2), {k:round(v,2) for k,v in d['kernels_ms_per_step'].items()})"
done > $O/r3b.log 2>&1
FXG_LIB=lib_alt/mask_glcm4/libfxg.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_scale_parity.py tests/test_batch.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -1 >> $O/r3b.log
cat $O/r3b.log
