cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1200 python -m pytest tests/test_batch.py tests/test_random_parity.py -m gpu -q -p no:cacheprovider -x -k "banded or packed or stack" 2>&1 | tail -2
: > $O/r5h.log
for i in 1 2 3; do
  FXG_PACK_TRACE=0 CALLS=9 timeout 300 python tools/pack_trace.py 2>&1 | grep "^call [345678]" | tr '\n' ' ' >> $O/r5h.log; echo >> $O/r5h.log
done
cat $O/r5h.log
CALLS=5 timeout 300 python tools/pack_trace.py 2>&1 | awk '/call 3:/{f=1} f' | grep "device\|call" | head -12
