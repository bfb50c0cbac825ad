cd $GRAFT_REPO_ROOT
O=gpurun_out
: > $O/r5i.log
for i in 1 2 3; do
for m in 1 0; do
  echo -n "merge $m: " >> $O/r5i.log
  FXG_PACK_MERGE=$m FXG_PACK_TRACE=0 CALLS=12 timeout 300 python tools/pack_trace.py 2>&1 | grep "^call" | tail -8 | awk '{s+=$3; n++} END {printf "%.3f ms avg of %d\n", s/n, n}' >> $O/r5i.log
done
done
cat $O/r5i.log
