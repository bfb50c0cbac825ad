"""Randomised parity sweep: many small seeded cases, each a random mix of mask
layout, intensity law and texture parameters, every group, device vs the oracle
(itself pinned bit for bit to the reference).  Complements the named-shape tests
with combinations nobody picked by hand: odd sizes, ng from 2 to 2000 (both
texture paths and the wide kernel), asymmetric GLCMs, 1-4 angles with
duplicates, offsets 1-3, histogram bins 1-1000.  The same cases also go
through the batch call (8 images per call), the banded host-raster path (64-row
bands) and the multi-context slide path (bands dealt over 3 contexts).
"""
import os

import numpy as np
import pytest

import inputs
from parity import assert_parity

import paper_2603_12016_b200 as fx
from oracle import make_params as oparams
from tools import synth

pytestmark = pytest.mark.gpu

ALL = ["intensity", "shape", "moments", "glcm", "glrlm", "glszm", "ngtdm"]


def _case(seed):
    rng = np.random.default_rng(1000 + seed)
    h, w = int(rng.integers(8, 160)), int(rng.integers(8, 160))
    kind = seed % 4
    if kind == 0:
        L = inputs.random_blobs((h, w), int(rng.integers(1, 25)), seed=seed,
                                max_r=int(rng.integers(2, 20)))
    elif kind == 1:
        L = inputs.random_labels((h, w), int(rng.integers(1, 12)), seed=seed,
                                 p_bg=float(rng.uniform(0.1, 0.9)))
    elif kind == 2:  # stripes and single pixels
        L = np.zeros((h, w), np.uint16)
        for k in range(int(rng.integers(1, 8))):
            y = int(rng.integers(0, h))
            L[y, : int(rng.integers(1, w + 1))] = k + 1
        L[rng.random((h, w)) < 0.01] = 60000
    else:  # blobs with scattered label values up to 65535
        vals = rng.choice(np.arange(1, 65536), size=6, replace=False)
        L = inputs.random_blobs((h, w), 12, seed=seed, max_r=15, label_values=vals)
    law = (seed // 4) % 5
    if law == 0:
        I = inputs.uniform((h, w), seed)
    elif law == 1:
        I = np.full((h, w), int(rng.integers(0, 65536)), np.uint16)
    elif law == 2:
        I = rng.integers(0, int(rng.integers(2, 12)), (h, w)).astype(np.uint16)
    elif law == 3:
        I = inputs.per_roi_levels(L, seed, noise=int(rng.integers(0, 200)))
    else:
        I = np.where(rng.random((h, w)) < 0.5, 0, 65535).astype(np.uint16)
    angles = tuple(int(a) for a in rng.choice([0, 45, 90, 135], size=int(rng.integers(1, 5))))
    over = dict(ng=int(rng.choice([2, 3, 16, 32, 64, 65, 100, 256, 257, 500, 2000])),
                offset=int(rng.integers(1, 4)), angles=angles,
                symmetric=bool(rng.integers(0, 2)),
                histogram_bins=int(rng.choice([1, 2, 7, 256, 1000])))
    return I, L, over


def _check(oracle, I, L, over, gl, gv):
    gp, op = fx.make_params("default", **over), oparams("default", **over)
    ol, ov = oracle.featurize(I, L, ALL, op)
    assert_parity(fx.feature_columns(ALL, gp), gl, gv, ol, ov, I, L)


# FX_RANDOM_CASES widens the sweep (e.g. 2000 for a bug hunt; 200 by default);
# FX_RANDOM_OFFSET starts every sweep at another seed
_OFF = int(os.environ.get("FX_RANDOM_OFFSET", "0"))


@pytest.mark.parametrize("seed", range(_OFF, _OFF + int(os.environ.get("FX_RANDOM_CASES", "200"))))
def test_random_case(ctx, oracle, seed):
    I, L, over = _case(seed)
    gl, gv = ctx.featurize(I, L, ALL, fx.make_params("default", **over))
    _check(oracle, I, L, over, gl, gv)


@pytest.mark.parametrize("k", range(_OFF, _OFF + int(os.environ.get("FX_RANDOM_BATCHES", "20"))))
def test_random_batch(ctx, oracle, k):
    cases = [_case(8 * k + j) for j in range(8)]
    over = cases[0][2]
    res = ctx.featurize_batch([(I, L) for I, L, _ in cases], ALL, fx.make_params("default", **over))
    for (I, L, _), (gl, gv) in zip(cases, res):
        _check(oracle, I, L, over, gl, gv)


@pytest.mark.parametrize("seed", range(_OFF, _OFF + int(os.environ.get("FX_RANDOM_BANDED", "40"))))
def test_random_banded(ctx, oracle, seed):
    I, L, over = _case(seed)
    try:
        ctx.set_band_rows(64)
        gl, gv = ctx.featurize(I, L, ALL, fx.make_params("default", **over))
    finally:
        ctx.set_band_rows(0)
    _check(oracle, I, L, over, gl, gv)


@pytest.fixture(scope="module")
def multi():
    m = fx.Multi([0, 0, 0])
    yield m
    m.close()


@pytest.mark.parametrize("seed", range(_OFF, _OFF + int(os.environ.get("FX_RANDOM_SLIDE", "40"))))
def test_random_slide(multi, oracle, seed):
    I, L, over = _case(seed)
    gl, gv = multi.featurize_slide(I, L, ALL, fx.make_params("default", **over))
    _check(oracle, I, L, over, gl, gv)


def _large_case(seed):
    """Bigger rasters (200-1100 px a side, up to a few hundred ROIs): every window
    class (S0/S1/S2, the CTA path, the texture kernel), many labels per warp tile
    of the scan, random profile and group subset."""
    rng = np.random.default_rng(5000 + seed)
    h, w = (int(v) for v in rng.integers(200, 1100, 2))
    kind = seed % 3
    if kind == 0:
        size = int(min(h, w))
        roi = int(rng.integers(20, 2500))
        pitch = int(np.ceil(3.8 * 1.1 * np.sqrt(roi / np.pi))) + 5  # the generator's grid pitch
        per_row = max(1, size // pitch)
        L = synth.blob_mask_grid(size, roi, int(rng.integers(1, per_row * per_row + 1)),
                                 int(rng.integers(1, 99)))
    elif kind == 1:
        vals = None
        if rng.random() < 0.5:
            vals = rng.choice(np.arange(1, 65536), size=int(rng.integers(2, 400)), replace=False)
        L = inputs.random_blobs((h, w), int(rng.integers(20, 400)), seed=seed,
                                max_r=int(rng.integers(3, 60)), label_values=vals)
    else:
        L = inputs.random_labels((h, w), int(rng.integers(2, 40)), seed=seed,
                                 p_bg=float(rng.uniform(0.3, 0.97)))
    law = int(rng.integers(0, 3))
    if law == 0:
        I = inputs.uniform(L.shape, seed)
    elif law == 1:
        I = inputs.per_roi_levels(L, seed, noise=int(rng.integers(0, 3000)))
    else:
        I = rng.integers(0, int(rng.integers(2, 70000)), L.shape).clip(0, 65535).astype(np.uint16)
    profile = str(rng.choice(["default", "performance", "ibsi-like"]))
    groups = [g for g in ALL if rng.random() < 0.6] or ["intensity"]
    angles = tuple(int(a) for a in rng.choice([0, 45, 90, 135], size=int(rng.integers(1, 5))))
    over = dict(ng=int(rng.choice([2, 8, 16, 32, 64, 100, 256, 300])),
                offset=int(rng.integers(1, 4)), angles=angles,
                symmetric=bool(rng.integers(0, 2)),
                histogram_bins=int(rng.choice([1, 16, 256, 1000])))
    return I, L, profile, groups, over


@pytest.mark.parametrize("seed", range(_OFF, _OFF + int(os.environ.get("FX_RANDOM_LARGE", "40"))))
def test_random_large(ctx, oracle, seed):
    I, L, profile, groups, over = _large_case(seed)
    gp, op = fx.make_params(profile, **over), oparams(profile, **over)
    gl, gv = ctx.featurize(I, L, groups, gp)
    ol, ov = oracle.featurize(I, L, groups, op)
    assert_parity(fx.feature_columns(groups, gp), gl, gv, ol, ov, I, L)


# window sizes at the class boundaries: S0 (<= 33 x 40 with the 40-wide stage),
# S1/S2 (<= 64 x 64), the 62-column fast-path limit, 64-row windows, L beyond
BOUNDARY_WINDOWS = [(33, 40), (34, 40), (33, 41), (62, 64), (63, 64), (64, 64), (64, 63), (64, 62),
                    (65, 64), (64, 65), (32, 64), (64, 32), (1, 64), (64, 1), (2, 2)]


@pytest.mark.parametrize("wh", BOUNDARY_WINDOWS, ids=[f"{w}x{h}" for w, h in BOUNDARY_WINDOWS])
@pytest.mark.parametrize("seed", range(_OFF, _OFF + int(os.environ.get("FX_RANDOM_BOUNDARY", "6"))))
def test_random_boundary_windows(ctx, oracle, wh, seed):
    """ROIs whose bounding box is exactly w x h: random fill (several components,
    holes) with pixels forced on all four box edges, placed at a random offset
    next to a second ROI; every group against the oracle."""
    w, h = wh
    rng = np.random.default_rng(7000 + 97 * seed + w * 131 + h)
    H, W = h + int(rng.integers(2, 20)), w + int(rng.integers(2, 20))
    L = np.zeros((H, W), np.uint16)
    y0, x0 = int(rng.integers(0, H - h + 1)), int(rng.integers(0, W - w + 1))
    box = rng.random((h, w)) < float(rng.uniform(0.2, 0.95))
    box[0, int(rng.integers(0, w))] = box[-1, int(rng.integers(0, w))] = True
    box[int(rng.integers(0, h)), 0] = box[int(rng.integers(0, h)), -1] = True
    lab = int(rng.choice([1, 77, 65535]))
    L[y0:y0 + h, x0:x0 + w] = np.where(box, lab, 0)
    free = L == 0
    L[free & (rng.random((H, W)) < 0.05)] = 3 if lab != 3 else 4  # a scattered second ROI
    I = rng.integers(0, int(rng.choice([4, 300, 65536])), (H, W)).astype(np.uint16)
    over = dict(ng=int(rng.choice([8, 64, 256, 300])), angles=(0, 45, 90, 135),
                symmetric=bool(rng.integers(0, 2)), offset=int(rng.integers(1, 3)))
    gp, op = fx.make_params("default", **over), oparams("default", **over)
    gl, gv = ctx.featurize(I, L, ALL, gp)
    ol, ov = oracle.featurize(I, L, ALL, op)
    assert_parity(fx.feature_columns(ALL, gp), gl, gv, ol, ov, I, L)


def test_random_small_masks_edge_sets(ctx, oracle):
    """SURVEY A1 at scale: random one-label masks of 3..12 x 3..12 pixels (fill
    0.3-0.9: several components, holes, border contact), batched; every group of
    every mask against the oracle (the edge set drives the edge statistics and
    the perimeter)."""
    n = int(os.environ.get("FX_RANDOM_SMALL", "2000"))
    rng = np.random.default_rng(4242 + _OFF)
    pairs = []
    for _ in range(n):
        h, w = (int(v) for v in rng.integers(3, 13, 2))
        m = rng.random((h, w)) < float(rng.uniform(0.3, 0.9))
        if not m.any():
            m[h // 2, w // 2] = True
        pad = int(rng.integers(0, 3))
        L = np.zeros((h + 2 * pad, w + 2 * pad), np.uint16)
        L[pad:pad + h, pad:pad + w] = m.astype(np.uint16) * int(rng.integers(1, 65536))
        I = rng.integers(0, 65536, L.shape).astype(np.uint16)
        pairs.append((I, L))
    p, op = fx.make_params("default"), oparams("default")
    cols = fx.feature_columns(ALL, p)
    res = ctx.featurize_batch(pairs, ALL, p)
    for (I, L), (gl, gv) in zip(pairs, res):
        ol, ov = oracle.featurize(I, L, ALL, op)
        assert_parity(cols, gl, gv, ol, ov, I, L)


@pytest.mark.parametrize("seed", range(_OFF, _OFF + int(os.environ.get("FX_RANDOM_ORIGIN", "30"))))
def test_random_device_pitch_origin(ctx, oracle, seed):
    """Device-resident rasters with a row pitch above the width and a tile origin:
    the table equals the reference's on the tile placed at that origin of a larger
    zero image (every coordinate column is global)."""
    import torch
    I, L, over = _case(seed)
    rng = np.random.default_rng(9000 + seed)
    h, w = L.shape
    ox, oy = int(rng.integers(0, 200)), int(rng.integers(0, 200))
    pitch = w + int(rng.integers(0, 40))
    gp, op = fx.make_params("default", **over), oparams("default", **over)
    cols = fx.feature_columns(ALL, gp)
    dI = torch.zeros((h, pitch), dtype=torch.int16, device="cuda")
    dL = torch.zeros((h, pitch), dtype=torch.int16, device="cuda")
    dI[:, :w] = torch.from_numpy(I.view(np.int16)).cuda()
    dL[:, :w] = torch.from_numpy(L.view(np.int16)).cuda()
    dL[:, w:] = 5  # garbage past the width: never read
    cap = int(np.count_nonzero(np.bincount(L.ravel(), minlength=65536)[1:])) + 1
    ol_ = torch.empty(cap, dtype=torch.int32, device="cuda")
    ov_ = torch.empty((cap, len(cols)), dtype=torch.float64, device="cuda")
    n = ctx.featurize_device(dI.data_ptr(), dL.data_ptr(), w, h, pitch, fx.resolve_groups(ALL), gp,
                             ol_.data_ptr(), ov_.data_ptr(), cap, origin=(ox, oy))
    torch.cuda.synchronize()
    gl = ol_[:n].cpu().numpy().view(np.uint32)
    gv = ov_[:n].cpu().numpy()
    Ib = np.zeros((h + oy, w + ox), np.uint16)
    Lb = np.zeros((h + oy, w + ox), np.uint16)
    Ib[oy:, ox:], Lb[oy:, ox:] = I, L
    rl, rv = oracle.featurize(Ib, Lb, ALL, op)
    assert_parity(cols, gl, gv, rl, rv, Ib, Lb)


@pytest.mark.parametrize("offset", [0, 1, 4, 5, 7, 8, 9, 15, 16, 17, 31, 32, 33, 40, 63, 64, 65, 100, 300])
def test_glcm_offsets_up_to_beyond_windows(ctx, oracle, offset):
    """GLCM offsets from 1 to beyond every window (no pair at all for most ROIs),
    small and large windows, symmetric and not, all angles."""
    rng = np.random.default_rng(offset)
    L = inputs.random_blobs((150, 170), 30, seed=offset, max_r=int(rng.integers(4, 40)))
    L[140:, :] = np.where(L[140:, :] > 0, L[140:, :], 0)
    I = rng.integers(0, int(rng.choice([5, 70, 65536])), L.shape).astype(np.uint16)
    for sym in (True, False):
        over = dict(ng=int(rng.choice([8, 64, 256, 300])), offset=offset, angles=(0, 45, 90, 135),
                    symmetric=sym)
        gp, op = fx.make_params("default", **over), oparams("default", **over)
        gl, gv = ctx.featurize(I, L, ["glcm"], gp)
        ol, ov = oracle.featurize(I, L, ["glcm"], op)
        assert_parity(fx.feature_columns(["glcm"], gp), gl, gv, ol, ov, I, L)


def test_every_label_value_present(ctx, oracle):
    """(Nearly) all 65,535 label values in one image: the label table's full range,
    ROIs of 1-4 pixels, labels in random order; every group against the oracle."""
    rng = np.random.default_rng(65535)
    # 2 x 2 cells of a 256 x 256 grid, labels in random order, one cell empty; some
    # cells lose pixels (ROIs of 1-4 pixels, diagonal-only contacts)
    grid = np.zeros(65536, np.uint16)
    grid[rng.permutation(65536)[:65535]] = np.arange(1, 65536, dtype=np.uint16)
    L = np.kron(grid.reshape(256, 256), np.ones((2, 2), np.uint16)).astype(np.uint16)
    L[rng.random(L.shape) < 0.2] = 0
    for lab in (1, 65535, 40000):  # keep a few labels present for the count check
        ys, xs = np.nonzero(np.kron(grid.reshape(256, 256) == lab, np.ones((2, 2), bool)))
        L[ys[0], xs[0]] = lab
    I = rng.integers(0, 65536, L.shape).astype(np.uint16)
    p, op = fx.make_params("default"), oparams("default")
    gl, gv = ctx.featurize(I, L, ALL, p)
    ol, ov = oracle.featurize(I, L, ALL, op)
    assert len(gl) == len(np.unique(L)) - 1 > 60000
    assert_parity(fx.feature_columns(ALL, p), gl, gv, ol, ov, I, L)
