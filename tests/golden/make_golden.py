"""Regenerates tests/golden/*.npz from the compiled reference (oracle/_ref).

Run in the build container (needs /root/reference to have been compiled into
oracle/_ref/libfxref.so):   python tests/golden/make_golden.py
Fixtures: inputs + the reference's own outputs, so the GPU box (which has no
/root/reference) can check the oracle and the device path against them.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))
import inputs  # noqa: E402
from oracle import Reference, make_params  # noqa: E402

GROUPS = ["intensity", "moments", "glcm"]


def main():
    ref = Reference()
    cases = {}
    L = ref.blob_mask_grid(192, 250, 16, 3)
    cases["blobs_uniform"] = (inputs.uniform(L.shape, 11), L)
    cases["blobs_star"] = (ref.siemens_star(192), L)
    cases["random_blobs"] = (inputs.uniform((80, 96), 5), inputs.random_blobs((80, 96), 25, seed=8))
    for k, m in inputs.adversarial_masks().items():
        cases["adv_" + k] = (inputs.uniform(m.shape, 2), m)
    for name, (I, L) in cases.items():
        out = {"intensity": I, "labels": L}
        for prof in ("default", "performance", "ibsi-like"):
            p = make_params(prof)
            rl, rv = ref.featurize(I, L, GROUPS, p, threads=1)
            out[f"{prof}_labels"] = rl
            out[f"{prof}_values"] = rv
            out[f"{prof}_columns"] = np.array(ref.columns(GROUPS, p))
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
        print(name, L.shape, len(out["default_labels"]))


if __name__ == "__main__":
    main()
