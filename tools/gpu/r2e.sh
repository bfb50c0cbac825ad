cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/r2e_pytest.log 2>&1; echo "rc=$?" >> $O/r2e_pytest.log
timeout 300 python tools/pcie_probe.py > $O/r2e_pcie.json 2> $O/r2e_pcie.err
tail -3 $O/r2e_pytest.log; cat $O/r2e_pcie.json
