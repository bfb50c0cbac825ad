cd $GRAFT_REPO_ROOT
O=gpurun_out
for rep in 1 2; do for v in "" lib_alt/flood32; do FXG_LIB=${v:+$v/libfxg.so} timeout 120 python tools/kbench.py c2 40 2>&1 | tail -1 | sed "s|^|${v:-default} |"; done; done > $O/r2z.log
FXG_LIB=lib_alt/flood32/libfxg.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_scale_parity.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -1 >> $O/r2z.log
cat $O/r2z.log
