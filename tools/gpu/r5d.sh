cd $GRAFT_REPO_ROOT
FX_RANDOM_SMALL=40000 timeout 1800 python -m pytest tests/test_random_parity.py -m gpu -q -p no:cacheprovider -k "small_masks" 2>&1 | grep -E "passed|failed|^E " | cut -c1-400 | head
