"""Shape group: device vs oracle on S-class inputs, per column worst ratio."""
import sys
import numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import inputs  # noqa: E402
import paper_2603_12016_b200 as fx  # noqa: E402
from oracle import Oracle, make_params  # noqa: E402
from parity import compare  # noqa: E402
ctx, o = fx.Context(0), Oracle()
cases = {"c1": fx.blob_mask_grid(512, 300, 100, 7), "blobs": inputs.random_blobs((96, 130), 40, seed=1)}
cases.update({k: v for k, v in inputs.adversarial_masks().items()})
for name, L in cases.items():
    I = inputs.uniform(L.shape, 3)
    gp, op = fx.resolve_profile("default"), make_params("default")
    cols = fx.feature_columns(["shape"], gp)
    gl, gv = ctx.featurize(I, L, ["shape"], gp)
    ol, ov = o.featurize(I, L, ["shape"], op)
    assert np.array_equal(gl, ol)
    bad = [(c, int(np.sum(gv[:, k] != ov[:, k]))) for k, c in enumerate(cols) if np.any(gv[:, k] != ov[:, k])]
    print(name, L.shape, len(gl), "cols differing (bitwise):", bad[:12])
    for c, _ in bad[:3]:
        k = cols.index(c)
        r = np.nonzero(gv[:, k] != ov[:, k])[0][:3]
        print("   ", c, [(int(gl[i]), gv[i, k], ov[i, k]) for i in r])
