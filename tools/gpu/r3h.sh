cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1500 python -m pytest tests/test_random_parity.py tests/test_gpu_parity.py tests/test_shard.py tests/test_batch.py -m gpu -q -p no:cacheprovider > $O/r3h.log 2>&1; echo "rc=$?" >> $O/r3h.log
grep -E "^E +|passed|failed|FAILED" $O/r3h.log | cut -c1-300 | head -40
