cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 600 python tools/bench_c5.py --steps 3 --warmup 1 > $O/r3j_c5.json 2> $O/r3j_c5.err; echo "rc=$?" >> $O/r3j_c5.err
timeout 300 python tools/kbench.py c5 3 > $O/r3j.log 2>&1
timeout 600 python -m pytest tests/test_scale_parity.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "c5 or large" >> $O/r3j.log 2>&1
cat $O/r3j_c5.json; tail -3 $O/r3j_c5.err; tail -5 $O/r3j.log
