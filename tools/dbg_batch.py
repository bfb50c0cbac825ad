"""Determinism probe: repeated featurize of one image; which columns/ROIs differ."""
import sys
import numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import paper_2603_12016_b200 as fx  # noqa: E402
from test_batch import _pairs, GROUPS  # noqa: E402
p = fx.resolve_profile("default")
I, L = _pairs([(256, 256, 40)], seed=17)[0]
ctx = fx.Context(0)
cols = fx.feature_columns(GROUPS, p)
lab, cnt, bb = ctx.roi_table(I, L)
ref = ctx.featurize(I, L, GROUPS, p)
for it in range(6):
    g = ctx.featurize(I, L, GROUPS if it % 2 == 0 else GROUPS[2:], p)
    if it % 2:
        continue
    d = np.nonzero(g[1] != ref[1])
    rows = sorted(set(d[0].tolist()))
    print("iter", it, "ndiff", len(d[0]), "rows", rows[:8])
    for r in rows[:4]:
        w, h = bb[r][2] - bb[r][0] + 1, bb[r][3] - bb[r][1] + 1
        cs = sorted(set(cols[c] for rr, c in zip(*d) if rr == r))
        print("  label", lab[r], "win", w, h, "n", cnt[r], "cols", cs[:6], len(cs))
