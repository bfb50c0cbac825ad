cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 300 python tools/kbench.py c2 20 > $O/r4e.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_random_parity.py tests/test_scale_parity.py -m gpu -q -p no:cacheprovider -x -k "label_scan or evicted or random_case or c2" >> $O/r4e.log 2>&1
tail -3 $O/r4e.log; head -1 $O/r4e.log
