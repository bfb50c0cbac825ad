"""Profiling driver: C2 workload, device-resident, N featurize calls (default 2)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import bench
import paper_2603_12016_b200 as fx

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2
groups = sys.argv[2].split(",") if len(sys.argv) > 2 else bench.GROUPS
profile = sys.argv[3] if len(sys.argv) > 3 else "default"
I, L, _ = bench.workload(0)
h, w = L.shape
nr = int(np.count_nonzero(np.bincount(L.ravel(), minlength=65536)[1:]))
p = fx.resolve_profile(profile)
g = fx.resolve_groups(groups)
nc = len(fx.feature_columns(g, p))
ctx = fx.Context(0)
di = torch.from_numpy(I.view(np.int16).reshape(-1)).cuda()
dl = torch.from_numpy(L.view(np.int16).reshape(-1)).cuda()
do = torch.empty((nr, nc), dtype=torch.float64, device="cuda")
dol = torch.empty((nr,), dtype=torch.int32, device="cuda")
for _ in range(n):
    assert ctx.featurize_device(di.data_ptr(), dl.data_ptr(), w, h, w, g, p, dol.data_ptr(), do.data_ptr(), nr) == nr
torch.cuda.synchronize()
print("ok", nr, nc)
