cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 600 python tools/gpu/dbg_random.py 19 22 24 > $O/r3d.log 2>&1; echo "rc=$?" >> $O/r3d.log
tail -c 6000 $O/r3d.log
