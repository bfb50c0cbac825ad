cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/r2i_pytest.log 2>&1; echo "rc=$?" >> $O/r2i_pytest.log
timeout 300 python tools/kbench.py c2 20 > $O/r2i_kbench.log 2>&1
timeout 300 python tools/kbench.py c3 20 >> $O/r2i_kbench.log 2>&1
FXG_LIB=lib_alt/pt/libfxg.so timeout 300 python tools/phase_clocks.py c2 >> $O/r2i_kbench.log 2>&1
timeout 600 python tools/bench_c4.py --tiles 10000 --steps 3 > $O/r2i_c4.json 2> $O/r2i_c4.err
tail -3 $O/r2i_pytest.log; cat $O/r2i_kbench.log; head -c 300 $O/r2i_c4.json
