# round 2, call b: fp64 peak, scan tuning sweep, per-group / C3 / C4 / C5 artifacts, ncu captures
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/r2b_pytest.log 2>&1; echo "rc=$?" >> $O/r2b_pytest.log
./tools/fp64_peak > $O/r2b_fp64.log 2>&1
for v in lib_alt/scan_*; do FXG_LIB=$v/libfxg.so timeout 120 python tools/kbench.py c2 20 2>&1 | tail -1; done > $O/r2b_scan_sweep.log
timeout 600 python tools/bench_groups.py --steps 20 > $O/r2b_groups.jsonl 2> $O/r2b_groups.err
timeout 600 python tools/bench_c4.py --tiles 10000 --steps 5 > $O/r2b_c4.json 2> $O/r2b_c4.err
timeout 900 python tools/bench_c4.py --tiles 10000 --steps 3 --groups intensity,shape,moments,glcm,glrlm,glszm,ngtdm > $O/r2b_c4_all7.json 2> $O/r2b_c4_all7.err
timeout 900 python tools/bench_c5.py --steps 3 > $O/r2b_c5.json 2> $O/r2b_c5.err
# ncu: each command first runs plain (&&), then under ncu
C4S="python tools/bench_c4.py --tiles 512 --distinct 64 --steps 1 --warmup 1 --e2e-tiles 8 --groups intensity,shape,moments,glcm,glrlm,glszm,ngtdm"
NCU="ncu --set full --clock-control none --import-source on"
timeout 300 python tools/kbench.py c3 2 > $O/r2b_plain_c3.log 2>&1 && \
  timeout 600 $NCU -k regex:k_roi_s -s 3 -c 1 -o $O/r2b_c3_s0 python tools/kbench.py c3 2 > $O/r2b_ncu_c3.log 2>&1
timeout 300 $C4S > $O/r2b_plain_c4.log 2>&1 && \
  timeout 900 $NCU -k regex:"k_roi_t|k_shape_serial|k_roi_s|k_serial_stats" -s 6 -c 6 -o $O/r2b_c4_all $C4S > $O/r2b_ncu_c4.log 2>&1
C5_SIZE=16384 timeout 300 python tools/kbench.py c5 1 > $O/r2b_plain_c5.log 2>&1 && \
  C5_SIZE=16384 timeout 900 $NCU -k regex:k_roi_b -s 3 -c 1 -o $O/r2b_c5_b python tools/kbench.py c5 1 > $O/r2b_ncu_c5.log 2>&1
timeout 300 python tools/kbench.py c2 2 > $O/r2b_plain_c2.log 2>&1 && \
  timeout 600 $NCU -k regex:"k_label_scan|k_roi_s|k_serial_stats" -s 9 -c 3 -o $O/r2b_c2 python tools/kbench.py c2 2 > $O/r2b_ncu_c2.log 2>&1
# reports -> CSV here (the .ncu-rep files would exceed the 64 MiB copy-back limit)
for r in $O/r2b_*.ncu-rep; do
  [ -f "$r" ] || continue
  b=${r%.ncu-rep}
  ncu -i $r --page raw --csv > $b.raw.csv 2>/dev/null
  ncu -i $r --page details --csv > $b.details.csv 2>/dev/null
  ncu -i $r --page source --csv 2>/dev/null | gzip > $b.source.csv.gz
  rm -f $r
done
ls -la $O; du -sh $O
