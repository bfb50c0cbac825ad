cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_batch.py tests/test_shard.py -m gpu -q -p no:cacheprovider -x -k "label_scan or c1 or batch or band or slide" > $O/r2s_pytest.log 2>&1; echo "rc=$?" >> $O/r2s_pytest.log
for v in "" lib_alt/scanb4; do FXG_LIB=${v:+$v/libfxg.so} timeout 120 python tools/kbench.py c2 30 2>&1 | tail -1 | sed "s|^|${v:-default} |"; done > $O/r2s_kbench.log
timeout 300 python tools/kbench.py c2 2 > $O/r2s_plain.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_label_scan" -s 3 -c 1 -o $O/r2s_scan python tools/kbench.py c2 2 > $O/r2s_ncu.log 2>&1
for r in $O/r2s_*.ncu-rep; do [ -f "$r" ] || continue; b=${r%.ncu-rep}; ncu -i $r --page raw --csv > $b.raw.csv 2>/dev/null; rm -f $r; done
tail -3 $O/r2s_pytest.log; cat $O/r2s_kbench.log
