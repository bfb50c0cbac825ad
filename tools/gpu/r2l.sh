cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "wide" > $O/r2l_wide.log 2>&1; echo "rc=$?" >> $O/r2l_wide.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/r2l_pytest.log 2>&1; echo "rc=$?" >> $O/r2l_pytest.log
tail -30 $O/r2l_wide.log; tail -5 $O/r2l_pytest.log
