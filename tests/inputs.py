"""Deterministic synthetic inputs for the parity tests.

Generators are numpy-only (seeded), plus the product's blob_mask_grid /
siemens_star (checked identical to the reference's in test_synth.py).
"""
from __future__ import annotations

import numpy as np


def uniform(shape, seed=0):
    return np.random.default_rng(seed).integers(0, 65536, size=shape, dtype=np.uint16)


def per_roi_levels(labels, seed=0, noise=40):
    """tertiary intensities: per-ROI base level plus small noise (realistic GLCM sparsity)"""
    rng = np.random.default_rng(seed)
    base = rng.integers(1000, 60000, size=65536)
    img = base[labels] + rng.integers(-noise, noise + 1, size=labels.shape)
    return np.clip(img, 0, 65535).astype(np.uint16)


def random_labels(shape, n_labels, seed=0, p_bg=0.3):
    rng = np.random.default_rng(seed)
    lab = rng.integers(1, n_labels + 1, size=shape).astype(np.uint16)
    lab[rng.random(shape) < p_bg] = 0
    return lab


def random_blobs(shape, n, seed=0, max_r=12, label_values=None):
    """Overlapping random discs/rectangles; later ones overwrite (gives multi-
    component ROIs, holes, thin bridges and border contact)."""
    rng = np.random.default_rng(seed)
    h, w = shape
    lab = np.zeros(shape, np.uint16)
    yy, xx = np.mgrid[0:h, 0:w]
    vals = label_values if label_values is not None else np.arange(1, n + 1)
    for i in range(n):
        L = vals[i % len(vals)]
        cx, cy = rng.integers(-3, w + 3), rng.integers(-3, h + 3)
        r = rng.integers(1, max_r + 1)
        if rng.random() < 0.5:
            m = (xx - cx) ** 2 + (yy - cy) ** 2 <= r * r
        else:
            m = (np.abs(xx - cx) <= r) & (np.abs(yy - cy) <= rng.integers(0, r + 1))
        if rng.random() < 0.3:  # punch a hole
            m &= ~((xx - cx) ** 2 + (yy - cy) ** 2 <= (r // 3) ** 2)
        lab[m] = L
    return lab


def adversarial_masks():
    """Named small masks covering the edge cases of SURVEY.md 8(d)."""
    out = {}
    # two equal-size components of one label (row-major tie-break, contour.cpp:57-60)
    m = np.zeros((12, 14), np.uint16)
    m[2:5, 1:4] = 7
    m[7:10, 9:12] = 7
    out["tie_components"] = m
    # diagonal one-pixel bridge between two squares (8-connected)
    m = np.zeros((10, 10), np.uint16)
    m[1:4, 1:4] = 3
    m[4, 4] = 3
    m[5:8, 5:8] = 3
    out["diag_bridge"] = m
    # ring with a hole + an island inside the hole (island is a separate component)
    m = np.zeros((11, 11), np.uint16)
    m[1:10, 1:10] = 5
    m[3:8, 3:8] = 0
    m[5, 5] = 5
    out["ring_island"] = m
    # ROIs touching every image border, single pixels, labels 1 and 65535
    m = np.zeros((9, 13), np.uint16)
    m[0, :] = 1
    m[:, 0] = 1
    m[8, 5:13] = 65535
    m[4, 6] = 2
    m[2:7, 12] = 40000
    out["borders_singletons"] = m
    # spiral (long exterior / interior paths)
    m = np.zeros((21, 21), np.uint16)
    x, y, d = 0, 0, 0
    dirs = [(1, 0), (0, 1), (-1, 0), (0, -1)]
    seg = 20
    while seg > 0:
        for _ in range(2):
            dx, dy = dirs[d % 4]
            for _ in range(seg):
                if 0 <= x < 21 and 0 <= y < 21:
                    m[y, x] = 9
                x += dx
                y += dy
            d += 1
        seg -= 2
    out["spiral"] = m
    # checkerboard label (every pixel its own 8-connected diagonal chain)
    m = ((np.indices((16, 16)).sum(0) % 2) * 4).astype(np.uint16)
    out["checker"] = m
    # comb with one-pixel teeth and U shapes
    m = np.zeros((12, 20), np.uint16)
    m[1, 1:19] = 11
    m[1:10, 1:19:2] = 11
    m[10, 3:16] = 12
    m[6:10, 3] = 12
    m[6:10, 15] = 12
    out["comb"] = m
    return out
