cd $GRAFT_REPO_ROOT
O=gpurun_out
for v in lib_alt/scan_*; do FXG_LIB=$v/libfxg.so timeout 120 python tools/kbench.py c2 30 2>&1 | tail -1 | sed "s|^|$v |"; done > $O/r2u_scan.log
cat $O/r2u_scan.log
