cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests/test_batch.py -m gpu -q -p no:cacheprovider -x -k "packed or banded" 2>&1 | tail -3
: > $O/r3t.log
for raw in 10 15 20 25; do
  echo "raw% $raw" >> $O/r3t.log
  FXG_PACK_RAW=$raw FXG_PACK_TRACE=0 CALLS=9 timeout 300 python tools/pack_trace.py 2>&1 | grep "^call [345678]" | tr '\n' ' ' >> $O/r3t.log
  echo >> $O/r3t.log
done
cat $O/r3t.log
