cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests/test_engine_cpp.py tests/test_batch.py -m gpu -q -p no:cacheprovider > $O/r2g_pytest.log 2>&1; echo "rc=$?" >> $O/r2g_pytest.log
for w in c2 c3 c5; do FXG_LIB=lib_alt/pt/libfxg.so timeout 300 python tools/phase_clocks.py $w; done > $O/r2g_phases.log 2>&1
FXG_LIB=lib_alt/pt/libfxg.so FX_GROUPS=intensity,shape,moments,glcm,glrlm,glszm,ngtdm timeout 300 python tools/phase_clocks.py c4 256 >> $O/r2g_phases.log 2>&1
tail -3 $O/r2g_pytest.log; cat $O/r2g_phases.log
