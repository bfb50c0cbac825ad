cd $GRAFT_REPO_ROOT
timeout 300 python tools/gpu/dbg_edge.py 2>&1 | tail -6
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "two_components or adversarial or debug or large" 2>&1 | tail -3
FX_RANDOM_CASES=6000 timeout 2400 python -m pytest tests/test_random_parity.py -m gpu -q -p no:cacheprovider -k "random_case" 2>&1 | grep -E "passed|failed|FAILED|^E " | cut -c1-300 | head
