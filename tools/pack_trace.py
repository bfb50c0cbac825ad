"""Host timeline of one packed fx_featurize call on the C2 image (FXG_PACK_TRACE)."""
import os
import sys
import time
os.environ.setdefault("FXG_PACK_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import bench  # noqa: E402
import paper_2603_12016_b200 as fx  # noqa: E402
I, L, _ = bench.workload(0)
ctx = fx.Context(0)
p = fx.resolve_profile(bench.PROFILE)
mask = fx.resolve_groups(bench.GROUPS)
ncols = len(fx.feature_columns(mask, p))
h, w = L.shape
n = bench.ROI_COUNT
hI = torch.from_numpy(I.view(np.int16)).pin_memory()
hL = torch.from_numpy(L.view(np.int16)).pin_memory()
hv = torch.empty((n, ncols), dtype=torch.float64).pin_memory()
hl = torch.empty(n, dtype=torch.int32).pin_memory()
for k in range(int(os.environ.get("CALLS", "6"))):
    t0 = time.perf_counter()
    ctx.featurize_host_ptrs(hI.data_ptr(), hL.data_ptr(), w, h, mask, p, hl.data_ptr(), hv.data_ptr(), n)
    print(f"call {k}: {1e3 * (time.perf_counter() - t0):.3f} ms", file=sys.stderr, flush=True)
ctx.enable_timing(True)
ctx.reset_kernel_times()
ctx.featurize_host_ptrs(hI.data_ptr(), hL.data_ptr(), w, h, mask, p, hl.data_ptr(), hv.data_ptr(), n)
kt = ctx.kernel_times()
for k, v in sorted(kt.items(), key=lambda kv: -kv[1][0]):
    print(f"kernel {k:22s} {v[0]:.3f} ms  x{v[1]}", file=sys.stderr)
