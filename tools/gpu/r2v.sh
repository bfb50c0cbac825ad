cd $GRAFT_REPO_ROOT
O=gpurun_out
for rep in 1 2; do for v in lib_alt/scan_*; do FXG_LIB=$v/libfxg.so timeout 120 python tools/kbench.py c2 40 2>&1 | tail -1 | sed "s|^|$v |"; done; done > $O/r2v_scan.log
cat $O/r2v_scan.log
