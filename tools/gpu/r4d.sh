cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 300 python tools/kbench.py c2 20 > $O/r4d.log 2>&1
FXG_LIB=lib_alt/ptall/libfxg.so timeout 300 python tools/phase_clocks.py c2 >> $O/r4d.log 2>&1
cat $O/r4d.log
