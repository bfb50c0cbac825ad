cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_random_parity.py -m gpu -q -p no:cacheprovider -k "every_label" 2>&1 | grep -E "passed|failed|FAILED|^E " | cut -c1-300 | head -20
