"""Host turnaround of the C2 featurize call: event-timed steps with and without
per-kernel timing, the sum of kernel times, and host wall per call.
usage: python tools/host_gap.py [steps]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2603_12016_b200 as fx  # noqa: E402
from tools import synth  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
L, _ = synth.packed_blob_mask_grid(8192, 400, 50000, 1)
I = synth.uniform_u16(L.shape, 0)
p = fx.resolve_profile("default")
mask = fx.resolve_groups(["intensity", "moments"])
ncols = len(fx.feature_columns(mask, p))
dI = torch.from_numpy(I.view(np.int16)).cuda()
dL = torch.from_numpy(L.view(np.int16)).cuda()
cap = 50000
ol = torch.empty(cap, dtype=torch.int32, device="cuda")
ov = torch.empty((cap, ncols), dtype=torch.float64, device="cuda")
ctx = fx.Context(0)
stream = torch.cuda.current_stream()
ctx.set_stream(stream.cuda_stream)
h, w = L.shape
run = lambda: ctx.featurize_device(dI.data_ptr(), dL.data_ptr(), w, h, w, mask, p, ol.data_ptr(),
                                   ov.data_ptr(), cap)
for _ in range(5):
    run()
torch.cuda.synchronize()
for timing in (False, True):
    ctx.enable_timing(timing)
    ctx.reset_kernel_times()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(stream)
    for _ in range(steps):
        run()
    e1.record(stream)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / steps * 1e3
    ms = e0.elapsed_time(e1) / steps
    kt = ctx.kernel_times()
    ksum = sum(v[0] for v in kt.values()) / steps if kt else float("nan")
    print(f"timing={timing}: {ms:.4f} ms/step (events), wall {wall:.4f} ms/call, kernel sum {ksum:.4f} ms")
ctx.enable_timing(False)
