cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/r2q_pytest.log 2>&1; echo "rc=$?" >> $O/r2q_pytest.log
timeout 600 python tools/bench_c4.py --tiles 10000 --steps 3 > $O/r2q_c4.json 2> $O/r2q_c4.err
timeout 300 python tools/kbench.py c2 20 > $O/r2q_kbench.log 2>&1
tail -3 $O/r2q_pytest.log; head -c 400 $O/r2q_c4.json; cat $O/r2q_kbench.log
