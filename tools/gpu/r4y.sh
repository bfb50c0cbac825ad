cd $GRAFT_REPO_ROOT
O=gpurun_out
FX_RANDOM_CASES=0 FX_RANDOM_LARGE=500 FX_RANDOM_BATCHES=400 FX_RANDOM_BANDED=800 FX_RANDOM_SLIDE=800 timeout 2400 python -m pytest tests/test_random_parity.py -m gpu -q -p no:cacheprovider > $O/r4y.log 2>&1; echo "rc=$?" >> $O/r4y.log
grep -E "passed|failed|FAILED|^E " $O/r4y.log | cut -c1-300 | head -30
