"""C4-shaped batch featurize for ncu captures: T tiles of 512 x 512, ~100 blob
ROIs each, groups from FX_GROUPS (default all seven), default profile.
usage: python tools/prof_c4.py [tiles] [repeats]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_12016_b200 as fx  # noqa: E402
from tools import synth  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 256
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
groups = os.environ.get("FX_GROUPS", "*ALL*").split(",")
labs = [synth.packed_blob_mask_grid(512, 1000, 100, s)[0] for s in range(16)]
pairs = [(synth.uniform_u16((512, 512), t), labs[t % 16]) for t in range(T)]
ctx = fx.Context(0)
out = ctx.featurize_batch(pairs, groups, fx.resolve_profile("default"))
if reps > 1:
    ctx.enable_timing(True)
    ctx.reset_kernel_times()
    for _ in range(reps - 1):
        out = ctx.featurize_batch(pairs, groups, fx.resolve_profile("default"))
    kt = ctx.kernel_times()
    print(" ".join(f"{k}={v[0] / (reps - 1):.3f}ms" for k, v in sorted(kt.items())))
print(len(out), "tiles,", sum(len(l) for l, _ in out), "ROIs")
