cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=12 > $O/r2f_pytest.log 2>&1; echo "rc=$?" >> $O/r2f_pytest.log
timeout 600 python bench.py --steps 100 --warmup 5 > $O/r2f_bench.json 2> $O/r2f_bench.err
tail -25 $O/r2f_pytest.log; head -c 600 $O/r2f_bench.json
