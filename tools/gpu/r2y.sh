# final measurement pass (round 2)
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/r2y_pytest.log 2>&1; echo "rc=$?" >> $O/r2y_pytest.log
timeout 600 python bench.py > $O/r2y_bench.json 2> $O/r2y_bench.err
timeout 600 python bench.py --impl reference > $O/r2y_bench_ref.json 2> $O/r2y_bench_ref.err
timeout 300 python tools/pcie_probe.py > $O/r2y_pcie.json 2> $O/r2y_pcie.err
timeout 600 python tools/bench_groups.py --steps 20 > $O/r2y_groups.jsonl 2> $O/r2y_groups.err
timeout 600 python tools/bench_c4.py --tiles 10000 --steps 3 > $O/r2y_c4.json 2> $O/r2y_c4.err
timeout 900 python tools/bench_c4.py --tiles 10000 --steps 3 --groups intensity,shape,moments,glcm,glrlm,glszm,ngtdm > $O/r2y_c4_all7.json 2> $O/r2y_c4_all7.err
timeout 900 python tools/bench_c5.py --steps 3 > $O/r2y_c5.json 2> $O/r2y_c5.err
tail -3 $O/r2y_pytest.log
