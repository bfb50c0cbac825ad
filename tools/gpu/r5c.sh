cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 300 python tools/kbench.py c2 20 2>&1 | tail -1 | cut -c1-60,150-260
timeout 300 python tools/kbench.py c2 20 2>&1 | tail -1 | cut -c1-60,150-260
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_random_parity.py tests/test_scale_parity.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -2
