cd $GRAFT_REPO_ROOT
O=gpurun_out
: > $O/r5r.log
for i in 1 2; do
for t in 11 13 15; do
  echo -n "threads $t: " >> $O/r5r.log
  FXG_PACK_THREADS=$t FXG_PACK_TRACE=0 CALLS=12 timeout 300 python tools/pack_trace.py 2>&1 | grep "^call" | tail -8 | awk '{s+=$3; n++} END {printf "%.3f ms avg of %d\n", s/n, n}' >> $O/r5r.log
done
done
cat $O/r5r.log
