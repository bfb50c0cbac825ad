cd $GRAFT_REPO_ROOT
O=gpurun_out
: > $O/r5j.log
for i in 1 2; do
for r in 15 20 25 30 35; do
  echo -n "raw $r: " >> $O/r5j.log
  FXG_PACK_RAW=$r FXG_PACK_TRACE=0 CALLS=12 timeout 300 python tools/pack_trace.py 2>&1 | grep "^call" | tail -8 | awk '{s+=$3; n++} END {printf "%.3f ms avg of %d\n", s/n, n}' >> $O/r5j.log
done
done
cat $O/r5j.log
