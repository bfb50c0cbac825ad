cd $GRAFT_REPO_ROOT
O=gpurun_out
FXG_LIB=lib_alt/pt/libfxg.so timeout 300 python tools/phase_clocks.py c2 > $O/r3a_phases.log 2>&1
FXG_LIB=lib_alt/pt/libfxg.so FX_GROUPS=intensity,moments,glcm timeout 300 python tools/phase_clocks.py c4 256 >> $O/r3a_phases.log 2>&1
cat $O/r3a_phases.log
