cd $GRAFT_REPO_ROOT
FX_RANDOM_BOUNDARY=40 timeout 1800 python -m pytest tests/test_random_parity.py -m gpu -q -p no:cacheprovider -k "boundary" 2>&1 | grep -E "passed|failed|FAILED|^E " | cut -c1-300 | head -30
