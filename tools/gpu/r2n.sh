# final-ish measurement pass: bench, launch list, ncu of the C2 kernels, C4 all
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 600 python bench.py > $O/r2n_bench.json 2> $O/r2n_bench.err
timeout 600 python bench.py --impl reference --steps 200 --warmup 5 > $O/r2n_bench_ref.json 2> $O/r2n_bench_ref.err
timeout 900 python tools/bench_c4.py --tiles 10000 --steps 3 --groups intensity,shape,moments,glcm,glrlm,glszm,ngtdm > $O/r2n_c4_all7.json 2> $O/r2n_c4_all7.err
timeout 600 python tools/bench_groups.py --steps 20 > $O/r2n_groups.jsonl 2> $O/r2n_groups.err
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/r2n_plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/r2n_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/r2n_ncu_launch.log 2>&1
timeout 300 python tools/kbench.py c2 2 > $O/r2n_plain_c2.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_label_scan|k_roi_s|k_serial_stats" -s 9 -c 3 -o $O/r2n_c2 python tools/kbench.py c2 2 > $O/r2n_ncu_c2.log 2>&1
for r in $O/r2n_*.ncu-rep; do
  [ -f "$r" ] || continue
  b=${r%.ncu-rep}
  ncu -i $r --page raw --csv > $b.raw.csv 2>/dev/null
  ncu -i $r --page source --csv 2>/dev/null | gzip > $b.source.csv.gz
  rm -f $r
done
ls -la $O | tail -20
