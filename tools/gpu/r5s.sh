cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/r5s_pytest.log 2>&1; echo "rc=$?" >> $O/r5s_pytest.log
tail -2 $O/r5s_pytest.log
