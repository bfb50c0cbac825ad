cd $GRAFT_REPO_ROOT
O=gpurun_out
FX_RANDOM_OFFSET=700000 FX_RANDOM_CASES=30000 FX_RANDOM_LARGE=800 FX_RANDOM_BATCHES=800 FX_RANDOM_BANDED=2000 FX_RANDOM_SLIDE=2000 FX_RANDOM_BOUNDARY=100 FX_RANDOM_SMALL=150000 FX_RANDOM_ORIGIN=3000 timeout 3300 python -m pytest tests/test_random_parity.py -m gpu -q -p no:cacheprovider -k "not every_label" > $O/r5t.log 2>&1; echo "rc=$?" >> $O/r5t.log
grep -E "passed|failed|FAILED|^E " $O/r5t.log | cut -c1-300 | head -40
