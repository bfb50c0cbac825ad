cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1500 python -m pytest tests/test_random_parity.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "random_large" > $O/r3e.log 2>&1; echo "rc=$?" >> $O/r3e.log
grep -E "^E +|passed|failed|FAILED" $O/r3e.log | cut -c1-400 | head -30
