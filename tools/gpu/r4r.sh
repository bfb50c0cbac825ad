cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_batch.py -m gpu -q -p no:cacheprovider -k "packed or stack" 2>&1 | tail -4
