cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests/test_batch.py tests/test_engine_cpp.py -m gpu -q -p no:cacheprovider -x > $O/r2k_pytest.log 2>&1; echo "rc=$?" >> $O/r2k_pytest.log
timeout 300 python tools/pcie_probe.py > $O/r2k_pcie.json 2> $O/r2k_pcie.err
tail -3 $O/r2k_pytest.log; cat $O/r2k_pcie.json
