cd $GRAFT_REPO_ROOT
O=gpurun_out
FXG_LIB=lib_alt/ptall/libfxg.so timeout 300 python tools/phase_clocks.py c5 > $O/r3i.log 2>&1
timeout 300 python tools/kbench.py c5 3 >> $O/r3i.log 2>&1
cat $O/r3i.log
