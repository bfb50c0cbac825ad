cd $GRAFT_REPO_ROOT
O=gpurun_out
NCU="ncu --set full --clock-control none --import-source on"
CALLS=2 FXG_PACK_TRACE=0 timeout 300 python tools/pack_trace.py > $O/r4j_plain.log 2>&1 && \
  CALLS=2 FXG_PACK_TRACE=0 timeout 900 $NCU -k regex:"k_unpack_intensity" -s 40 -c 2 -o $O/r4j_unpack python tools/pack_trace.py > $O/r4j_ncu.log 2>&1
for r in $O/r4j_*.ncu-rep; do
  [ -f "$r" ] || continue
  b=${r%.ncu-rep}
  ncu -i $r --page raw --csv > $b.raw.csv 2>/dev/null
  ncu -i $r --page details --csv > $b.details.csv 2>/dev/null
  ncu -i $r --page source --csv 2>/dev/null | gzip > $b.source.csv.gz
  rm -f $r
done
ls $O/r4j*; tail -3 $O/r4j_ncu.log
