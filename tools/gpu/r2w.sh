cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/r2w_pytest.log 2>&1; echo "rc=$?" >> $O/r2w_pytest.log
timeout 600 python bench.py > $O/r2w_bench.json 2> $O/r2w_bench.err
timeout 300 python tools/kbench.py c2 2 > $O/r2w_plain.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_label_scan" -s 3 -c 1 -o $O/r2w_scan python tools/kbench.py c2 2 > $O/r2w_ncu.log 2>&1
for r in $O/r2w_*.ncu-rep; do [ -f "$r" ] || continue; b=${r%.ncu-rep}; ncu -i $r --page raw --csv > $b.raw.csv 2>/dev/null; rm -f $r; done
tail -3 $O/r2w_pytest.log; head -c 300 $O/r2w_bench.json
