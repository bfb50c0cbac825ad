"""Edge-set (trace_contour visited set) of one ROI: device vs oracle, on the
randomized case that disagreed, its window alone, and transformed copies."""
import sys
sys.path[:0] = ["tests", "."]
import numpy as np
import test_random_parity as t
import oracle
import paper_2603_12016_b200 as fx

O = oracle.Oracle()
ctx = fx.Context(0)
p = fx.make_params("default", histogram_bins=16)
I, L, _ = t._case(int(sys.argv[1]) if len(sys.argv) > 1 else 5203)
lab = int(sys.argv[2]) if len(sys.argv) > 2 else 63242


def check(name, I, L, lab):
    ys, xs = np.nonzero(L == lab)
    _, edge, _, _ = ctx.debug_roi(I, L, lab, p)
    pts = O.trace_contour(xs, ys)
    a, b = set(map(tuple, edge.tolist())), set(map(tuple, pts.tolist()))
    print(f"{name}: dev {len(a)} ref {len(b)} equal {a == b}; dev-only {sorted(a - b)[:6]} ref-only {sorted(b - a)[:6]}")


check("case", I, L, lab)
ys, xs = np.nonzero(L == lab)
win = (slice(ys.min(), ys.max() + 1), slice(xs.min(), xs.max() + 1))
Lw = np.where(L[win] == lab, lab, 0).astype(np.uint16)
check("window only", I[win].copy(), Lw, lab)
pad = np.zeros((Lw.shape[0] + 8, Lw.shape[1] + 8), np.uint16)
pad[4:-4, 4:-4] = Lw
check("window padded", np.zeros_like(pad), pad, lab)
check("flipped lr", I[win][:, ::-1].copy(), Lw[:, ::-1].copy(), lab)
check("flipped ud", I[win][::-1].copy(), Lw[::-1].copy(), lab)
check("transposed", I[win].T.copy(), Lw.T.copy(), lab)
