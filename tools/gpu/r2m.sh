cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "wide" > $O/r2m_wide.log 2>&1; echo "rc=$?" >> $O/r2m_wide.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/r2m_pytest.log 2>&1; echo "rc=$?" >> $O/r2m_pytest.log
grep -E "^E +Assert|passed|failed" $O/r2m_wide.log | cut -c1-600; tail -5 $O/r2m_pytest.log
