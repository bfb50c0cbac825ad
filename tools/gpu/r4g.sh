cd $GRAFT_REPO_ROOT
O=gpurun_out
C4S="python tools/bench_c4.py --tiles 512 --distinct 64 --steps 1 --warmup 1 --e2e-tiles 8 --groups intensity,shape,moments,glcm,glrlm,glszm,ngtdm"
NCU="ncu --set full --clock-control none --import-source on"
timeout 300 $C4S > $O/r4g_plain.log 2>&1 && \
  timeout 900 $NCU -k regex:"k_roi_t" -s 2 -c 1 -o $O/r4g_t $C4S > $O/r4g_ncu.log 2>&1
for r in $O/r4g_*.ncu-rep; do
  [ -f "$r" ] || continue
  b=${r%.ncu-rep}
  ncu -i $r --page raw --csv > $b.raw.csv 2>/dev/null
  ncu -i $r --page details --csv > $b.details.csv 2>/dev/null
  ncu -i $r --page source --csv 2>/dev/null | gzip > $b.source.csv.gz
  rm -f $r
done
ls -la $O/r4g*; tail -2 $O/r4g_ncu.log
