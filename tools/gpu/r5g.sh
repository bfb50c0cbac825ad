cd $GRAFT_REPO_ROOT
FX_RANDOM_ORIGIN=400 timeout 1500 python -m pytest tests/test_random_parity.py -m gpu -q -p no:cacheprovider -k "pitch_origin" 2>&1 | grep -E "passed|failed|FAILED|^E " | cut -c1-300 | head -20
