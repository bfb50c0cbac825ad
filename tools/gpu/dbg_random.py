"""Debug randomised parity cases: args 'seed' or 'seed:pseed' (image of seed,
parameters of pseed); prints the violating cells with both values."""
import sys
sys.path[:0] = ["tests", "."]
import numpy as np
import test_random_parity as t
import oracle
import paper_2603_12016_b200 as fx
from parity import floors, compare

np.set_printoptions(precision=17, linewidth=220)
O = oracle.Oracle()
ctx = fx.Context(0)
ALL = t.ALL
for arg in sys.argv[1:]:
    s, ps = (int(a) for a in arg.split(":")) if ":" in arg else (int(arg), int(arg))
    I, L, _ = t._case(s)
    o = t._case(ps)[2]
    gp, op = fx.make_params("default", **o), oracle.make_params("default", **o)
    cols = fx.feature_columns(ALL, gp)
    gl, gv = ctx.featurize(I, L, ALL, gp)
    ol, ov = O.featurize(I, L, ALL, op)
    print(f"== {arg} shape {L.shape} {o} labels-equal {np.array_equal(gl, ol)}")
    if not np.array_equal(gl, ol):
        continue
    sc = floors(cols, ov, I, L, np.asarray(ol))
    for i, c in enumerate(cols):
        bound = (1e-6 if c.startswith("glcm_") else 1e-9) * (np.maximum(abs(gv[:, i]), abs(ov[:, i])) + sc[:, i])
        rows = np.nonzero(~((abs(gv[:, i] - ov[:, i]) <= bound) | (gv[:, i] == ov[:, i])))[0]
        if c in ("shape_orientation",) or not len(rows):
            continue
        print(f"  col {i} {c}: {len(rows)} rows")
        for k in rows[:3]:
            lab = int(gl[k])
            ys, xs = np.nonzero(L == lab)
            vals = np.unique(I[ys, xs])
            print(f"  {c} row {k} label {lab} n={len(xs)} bbox x{xs.min()}-{xs.max()} y{ys.min()}-{ys.max()} "
                  f"levels {len(vals)}: dev {gv[k, i]!r} ref {ov[k, i]!r}")
            if len(xs) <= 40:
                print("    px", list(zip(xs.tolist(), ys.tolist())), "vals", I[ys, xs].tolist())
