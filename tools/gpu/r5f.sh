cd $GRAFT_REPO_ROOT
O=gpurun_out
FX_RANDOM_OFFSET=100000 FX_RANDOM_CASES=20000 FX_RANDOM_LARGE=600 FX_RANDOM_BATCHES=600 FX_RANDOM_BANDED=1500 FX_RANDOM_SLIDE=1500 FX_RANDOM_BOUNDARY=60 FX_RANDOM_SMALL=100000 timeout 3000 python -m pytest tests/test_random_parity.py -m gpu -q -p no:cacheprovider > $O/r5f.log 2>&1; echo "rc=$?" >> $O/r5f.log
grep -E "passed|failed|FAILED|^E " $O/r5f.log | cut -c1-300 | head -40
