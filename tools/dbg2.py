import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import inputs
import paper_2603_12016_b200 as fx
from oracle import Oracle, make_params as op
from parity import floors, compare
o = Oracle(); ctx = fx.Context(0)
L = inputs.adversarial_masks()["ring_island"]; I = inputs.uniform(L.shape, 3)
p = fx.make_params("default", histogram_bins=16)
hist, edge, glcm, pairs = ctx.debug_roi(I, L, 5, p)
ys, xs = np.nonzero(L == 5)
pts = o.trace_contour(xs, ys)
print("gpu edge", sorted(map(tuple, edge.tolist())))
print("ora edge", sorted(set(map(tuple, pts.tolist()))))
G = ["intensity", "moments", "glcm"]
Lb = fx.blob_mask_grid(256, 220, 25, 5); Ib = inputs.uniform(Lb.shape, 6)
for over in [dict(histogram_bins=2), dict(histogram_bins=1000), dict(offset=2), dict(ng=2), dict(ng=7, symmetric=False, angles=(135, 0, 45)), dict(angles=(90, 90))]:
    gp = fx.make_params("default", **over); opp = op("default", **over)
    gl, gv = ctx.featurize(Ib, Lb, G, gp); ol, ov = o.featurize(Ib, Lb, G, opp)
    cols = fx.feature_columns(G, gp)
    bad = compare(cols, gv, ov, floors(cols, ov, Ib, Lb, ol))
    print(over, [b[:2] for b in bad[:6]])
Lt = fx.blob_mask_grid(768, 600, 250, 3)
It = inputs.per_roi_levels(Lt, 5)
try:
    gl, gv = ctx.featurize(It, Lt, G, fx.make_params("default"))
    ol, ov = o.featurize(It, Lt, G, op("default"))
    cols = fx.feature_columns(G, fx.make_params("default"))
    bad = compare(cols, gv, ov, floors(cols, ov, It, Lt, ol))
    print("tertiary", [b for b in bad[:8]])
except Exception as e:
    print("tertiary ERR", e)
