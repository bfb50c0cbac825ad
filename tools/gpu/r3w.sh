cd $GRAFT_REPO_ROOT
O=gpurun_out
: > $O/r3w.log
for split in 0 1; do
for br in 0 1536 2048 3072 4096; do
  echo "split $split band_rows $br" >> $O/r3w.log
  FXG_PACK_SPLIT=$split FXG_BAND_ROWS=$br FXG_PACK_TRACE=0 CALLS=9 timeout 300 python tools/pack_trace.py 2>&1 | grep "^call [345678]" | tr '\n' ' ' >> $O/r3w.log
  echo >> $O/r3w.log
done
done
cat $O/r3w.log
