"""Per-kernel device times of one featurize workload (for A/B of library builds).
usage: FXG_LIB=... python tools/kbench.py [c2|c3] [steps]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2603_12016_b200 as fx  # noqa: E402
from tools import synth  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "c2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
if which == "c2":
    L, _ = synth.packed_blob_mask_grid(8192, 400, 50000, 1)
    groups = os.environ.get("FX_GROUPS", "intensity,moments").split(",")
    prof = "default"
elif which.startswith("c5"):  # C5 regime at reduced size: 16384^2, ~2e5-px blobs
    size = int(os.environ.get("C5_SIZE", "16384"))
    n = (size // 680) ** 2
    L, _ = synth.packed_blob_mask_grid(size, 200000, n, 1)
    groups = ["intensity", "moments", "glcm"]
    prof = "default"
else:  # c3: 4096^2, 10k ROIs, GLCM 4 angles ng=256
    L, _ = synth.packed_blob_mask_grid(4096, 400, 10000, 1)
    groups = ["glcm"]
    prof = "ibsi-like"
I = synth.uniform_u16(L.shape, 0)
law = os.environ.get("FX_LAW", "uniform")  # intensity law: uniform u16 | twelve (0..4095) | narrow
if law == "twelve":
    I = I & np.uint16(4095)
elif law == "narrow":
    I = (I % np.uint16(300) + np.uint16(1000)).astype(np.uint16)
p = fx.resolve_profile(prof)
mask = fx.resolve_groups(groups)
ncols = len(fx.feature_columns(mask, p))
dI = torch.from_numpy(I.view(np.int16)).cuda()
dL = torch.from_numpy(L.view(np.int16)).cuda()
cap = int(np.count_nonzero(np.bincount(L.ravel(), minlength=65536)[1:]))
ol = torch.empty(cap, dtype=torch.int32, device="cuda")
ov = torch.empty((cap, ncols), dtype=torch.float64, device="cuda")
ctx = fx.Context(0)
h, w = L.shape
run = lambda: ctx.featurize_device(dI.data_ptr(), dL.data_ptr(), w, h, w, mask, p, ol.data_ptr(),
                                   ov.data_ptr(), cap)
for _ in range(3):
    run()
ctx.enable_timing(True)
ctx.reset_kernel_times()
for _ in range(steps):
    run()
kt = ctx.kernel_times()
tot = sum(v[0] for v in kt.values()) / steps
lib = os.path.basename(os.environ.get("FXG_LIB", "lib/libfxg.so"))
print(f"{lib:24s} {which} total {tot:.4f} ms | " +
      " ".join(f"{k}={v[0] / steps:.4f}" for k, v in sorted(kt.items())))
