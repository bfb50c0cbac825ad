cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1500 python -m pytest tests/test_random_parity.py -m gpu -q -p no:cacheprovider > $O/r3f.log 2>&1; echo "rc=$?" >> $O/r3f.log
grep -E "^E +|passed|failed|FAILED" $O/r3f.log | cut -c1-300 | head -40
