"""Per-call latency of the per-ROI operator (fx_roi_features) and the per-cloud cost of
fx_roi_features_batch.  usage: python tools/roi_latency.py"""
import time, numpy as np, sys
sys.path.insert(0, '.')
import paper_2603_12016_b200 as fx
ctx = fx.Context(0)
rng = np.random.default_rng(0)
ys, xs = np.nonzero(np.hypot(*np.mgrid[-9:10, -9:10]) <= 9)
xs = (xs + 100).astype(np.uint32); ys = (ys + 200).astype(np.uint32)
vs = rng.integers(0, 65535, len(xs)).astype(np.uint16)
for groups in (["intensity"], ["intensity", "moments"], ["*ALL*"]):
    for _ in range(5): ctx.roi_features(xs, ys, vs, groups)
    t = time.perf_counter(); N = 300
    for _ in range(N): ctx.roi_features(xs, ys, vs, groups)
    print(groups, f"{(time.perf_counter() - t) / N * 1e6:.0f} us per call ({len(xs)} px)")
    clouds = [(xs, ys, vs)] * 10000
    ctx.roi_features_batch(clouds[:100], groups)
    t = time.perf_counter()
    ctx.roi_features_batch(clouds, groups)
    print(groups, f"batch of {len(clouds)}: {(time.perf_counter() - t) / len(clouds) * 1e6:.1f} us per cloud")
