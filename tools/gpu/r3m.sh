cd $GRAFT_REPO_ROOT
O=gpurun_out
NCU="ncu --set full --clock-control none --import-source on"
C5_SIZE=16384 timeout 300 python tools/kbench.py c5 1 > $O/r3m_plain_c5.log 2>&1 && \
  C5_SIZE=16384 timeout 900 $NCU -k regex:k_roi_b -s 3 -c 1 -o $O/r3m_c5_b python tools/kbench.py c5 1 > $O/r3m_ncu_c5.log 2>&1
for r in $O/r3m_*.ncu-rep; do
  [ -f "$r" ] || continue
  b=${r%.ncu-rep}
  ncu -i $r --page raw --csv > $b.raw.csv 2>/dev/null
  ncu -i $r --page details --csv > $b.details.csv 2>/dev/null
  ncu -i $r --page source --csv 2>/dev/null | gzip > $b.source.csv.gz
  ncu -i $r --page source --csv --print-source sass 2>/dev/null | gzip > $b.sass.csv.gz
  rm -f $r
done
tail -2 $O/r3m_plain_c5.log; ls -la $O/r3m*
