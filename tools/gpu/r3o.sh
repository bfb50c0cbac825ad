cd $GRAFT_REPO_ROOT
O=gpurun_out
FX_GROUPS=intensity,shape,moments,glcm,glrlm,glszm,ngtdm FXG_LIB=lib_alt/ptall/libfxg.so timeout 300 python tools/phase_clocks.py c4 512 > $O/r3o.log 2>&1
cat $O/r3o.log
