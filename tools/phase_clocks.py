"""Per-phase clock shares of the S-class ROI kernels (phase-timing build).
usage: FXG_LIB=.../libfxg_pt.so python tools/phase_clocks.py c2|c3|c4|c5 [tiles]"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_12016_b200 as fx  # noqa: E402
from tools import synth  # noqa: E402
from paper_2603_12016_b200 import fxg  # noqa: E402

NAMES = ["load+gather", "int sort", "int stats", "edge", "moments", "glcm keys", "glcm sort",
         "glcm rle", "haralick"]
BNAMES = ["B words+scan", "B pixels", "B int hist/order", "B edge+int out", "B moments",
          "B glcm levels", "B glcm angles"]
which = sys.argv[1]
ctx = fx.Context(0)
lib = fxg.lib()
buf = (C.c_ulonglong * 16)()
if which == "c2":
    L, _ = synth.packed_blob_mask_grid(8192, 400, 50000, 1)
    I = synth.uniform_u16(L.shape, 0)
    run = lambda: ctx.featurize(I, L, ["intensity", "moments"], fx.resolve_profile("default"))
    nroi = 50000
elif which == "c4":
    T = int(sys.argv[2]) if len(sys.argv) > 2 else 256
    pairs = []
    for t in range(T):
        Lt, _ = synth.packed_blob_mask_grid(512, 1000, 100, t % 16)
        pairs.append((synth.uniform_u16(Lt.shape, t), Lt))
    groups = os.environ.get("FX_GROUPS", "intensity,moments,glcm").split(",")
    run = lambda: ctx.featurize_batch(pairs, groups, fx.resolve_profile("default"))
    nroi = sum(int(np.count_nonzero(np.bincount(p[1].ravel(), minlength=65536)[1:])) for p in pairs)
if which == "c3":
    L, _ = synth.packed_blob_mask_grid(4096, 400, 10000, 1)
    I = synth.uniform_u16(L.shape, 0)
    run = lambda: ctx.featurize(I, L, ["glcm"], fx.resolve_profile("ibsi-like"))
    nroi = 10000
if which == "c5":
    L, _ = synth.packed_blob_mask_grid(16384, 200000, 576, 1)
    I = synth.uniform_u16(L.shape, 0)
    run = lambda: ctx.featurize(I, L, ["intensity", "moments", "glcm"], fx.resolve_profile("default"))
    nroi = int(L.max())
tbuf = (C.c_ulonglong * 8)()
run()
lib.fx_debug_phase_clocks(buf, 16, 1)
lib.fx_debug_texture_clocks(tbuf, 8, 1)
run()
assert lib.fx_debug_phase_clocks(buf, 16, 1) == 0, "not a phase-timing build"
lib.fx_debug_texture_clocks(tbuf, 8, 1)
tot = sum(buf[:9])
print(f"{which}: {nroi} ROIs, {tot / nroi:.0f} clocks per ROI (lane 0, S kernels)")
for k, nm in enumerate(NAMES):
    print(f"  {nm:12s} {buf[k] / nroi:9.0f} clk/ROI  {100 * buf[k] / max(tot, 1):5.1f}%")
totb = sum(buf[9:16])
if totb:
    print(f"large-ROI kernel: {totb / nroi:.0f} clocks per ROI (thread 0)")
    for k, nm in enumerate(BNAMES):
        print(f"  {nm:16s} {buf[9 + k] / nroi:10.0f} clk/ROI  {100 * buf[9 + k] / totb:5.1f}%")
tt = sum(tbuf[:4]) + tbuf[7]  # slots 4-6 split GLRLM (slot 1), 7 is GLSZM's zones
if tt:
    names = ["discretize", "GLRLM other", "GLSZM", "NGTDM", "GLRLM runs", "GLRLM features",
             "GLRLM restore", "GLSZM zones"]
    print(f"texture kernel: {tt / nroi:.0f} clocks per ROI (thread 0)")
    for k, nm in enumerate(names):
        print(f"  {nm:16s} {tbuf[k] / nroi:10.0f} clk/ROI  {100 * tbuf[k] / tt:5.1f}%")
