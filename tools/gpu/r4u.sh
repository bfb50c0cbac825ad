cd $GRAFT_REPO_ROOT
O=gpurun_out
FX_RANDOM_CASES=3000 FX_RANDOM_LARGE=200 timeout 2400 python -m pytest tests/test_random_parity.py -m gpu -q -p no:cacheprovider -k "random_case or random_large" > $O/r4u.log 2>&1; echo "rc=$?" >> $O/r4u.log
grep -E "passed|failed|FAILED|^E " $O/r4u.log | cut -c1-300 | head -30
