cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1500 python -m pytest tests/test_random_parity.py -m gpu -q -p no:cacheprovider > $O/r3c.log 2>&1; echo "rc=$?" >> $O/r3c.log
grep -E "^E +Assert|passed|failed|FAILED" $O/r3c.log | cut -c1-400 | head -30
