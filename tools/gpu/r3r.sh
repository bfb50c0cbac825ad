cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 300 python tools/pack_trace.py > $O/r3r.log 2>&1
grep -v "intensity packed\|labels packed" $O/r3r.log | tail -26; grep "packed" $O/r3r.log | tail -66 | awk 'NR%6==0'
