cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_scale_parity.py -m gpu -q -p no:cacheprovider -x > $O/r2h_pytest.log 2>&1; echo "rc=$?" >> $O/r2h_pytest.log
timeout 300 python tools/kbench.py c3 20 > $O/r2h_kbench.log 2>&1
FXG_LIB=lib_alt/pt/libfxg.so timeout 300 python tools/phase_clocks.py c3 >> $O/r2h_kbench.log 2>&1
tail -3 $O/r2h_pytest.log; cat $O/r2h_kbench.log
