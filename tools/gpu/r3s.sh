cd $GRAFT_REPO_ROOT
O=gpurun_out


timeout 300 python tools/pack_trace.py > $O/r3s_trace.log 2>&1
grep -v "intensity packed\|labels packed" $O/r3s_trace.log | tail -60
