cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/r2d_pytest.log 2>&1; echo "rc=$?" >> $O/r2d_pytest.log
timeout 300 python tools/pcie_probe.py > $O/r2d_pcie.json 2> $O/r2d_pcie.err
timeout 300 python tools/kbench.py c2 20 > $O/r2d_kbench.log 2>&1
tail -3 $O/r2d_pytest.log; cat $O/r2d_pcie.json $O/r2d_kbench.log
