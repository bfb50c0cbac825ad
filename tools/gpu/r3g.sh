cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 600 python tools/gpu/dbg_random.py 5203 3748 > $O/r3g.log 2>&1
grep -v "^== .*labels-equal True$" $O/r3g.log | cut -c1-700 | head -80
