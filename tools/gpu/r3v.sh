cd $GRAFT_REPO_ROOT
O=gpurun_out
CALLS=5 timeout 300 python tools/pack_trace.py > $O/r3v.log 2>&1
awk '/call 3:/{f=1} f' $O/r3v.log | grep -v "^kernel" | head -80
