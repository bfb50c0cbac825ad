cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_scale_parity.py -m gpu -q -p no:cacheprovider -x > $O/r2j_pytest.log 2>&1; echo "rc=$?" >> $O/r2j_pytest.log
timeout 300 python tools/kbench.py c2 20 > $O/r2j_kbench.log 2>&1
timeout 300 python tools/kbench.py c3 20 >> $O/r2j_kbench.log 2>&1
timeout 600 python tools/bench_c4.py --tiles 10000 --steps 3 > $O/r2j_c4.json 2> $O/r2j_c4.err
tail -3 $O/r2j_pytest.log; cat $O/r2j_kbench.log; head -c 300 $O/r2j_c4.json
