cd $GRAFT_REPO_ROOT
timeout 300 python tools/gpu/dbg_edge.py 2>&1 | tail -8
