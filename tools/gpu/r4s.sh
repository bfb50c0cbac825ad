# round-2 final measurement pass: bench, reference arm, launch list, ncu of the C2 kernels
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 600 python bench.py > $O/r4s_bench.json 2> $O/r4s_bench.err
timeout 600 python bench.py --impl reference --steps 200 --warmup 5 > $O/r4s_bench_ref.json 2> $O/r4s_bench_ref.err
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/r4s_plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/r4s_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/r4s_ncu_launch.log 2>&1
timeout 300 python tools/kbench.py c2 2 > $O/r4s_plain_c2.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_label_scan|k_roi_s|k_serial_stats" -s 9 -c 3 -o $O/r4s_c2 python tools/kbench.py c2 2 > $O/r4s_ncu_c2.log 2>&1
for r in $O/r4s_*.ncu-rep; do
  [ -f "$r" ] || continue
  b=${r%.ncu-rep}
  ncu -i $r --page raw --csv > $b.raw.csv 2>/dev/null
  ncu -i $r --page source --csv 2>/dev/null | gzip > $b.source.csv.gz
  rm -f $r
done
ls -la $O | tail -20
