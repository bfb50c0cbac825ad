"""GPU parity at BASELINE.json's named config shapes (north_star).

Each test featurizes one of the benchmark workloads at its full size through the
C ABI and compares the whole table with the reference's own CPU path
(oracle/_ref: /root/reference/proj/src compiled unmodified, accumulate +
compute_roi_features per label, engine.cpp:300-333) -- or, where that library
was not built, with the C restatement pinned bit for bit to it.

  C2  8192^2, 50k ROIs, intensity + moments     -- exactly bench.py's workload(0)
  C3  4096^2, 10k ROIs, GLCM ibsi-like (ng 256)  -- the sort path
  C4  a full 512-slot launch set of 512^2 tiles, *ALL* groups (fx_featurize_batch)
  C5  16384^2 slide, ~2e5-px ROIs (large-ROI CTA kernel), intensity+moments+glcm

These are the code paths that only occur at scale: the staging bump allocators
with 50k ROIs, class lists of tens of thousands, the S->L overflow re-queue and
the persistent large-ROI kernel.
"""
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from parity import assert_parity

import paper_2603_12016_b200 as fx
from tools import synth
import oracle as O

pytestmark = pytest.mark.gpu

ALL = ["intensity", "shape", "moments", "glcm", "glrlm", "glszm", "ngtdm"]


def _checker():
    """(featurize(I, L, groups, params, threads), params factory) of the reference
    library when present, else of the C restatement (pinned to it bitwise)."""
    if O.reference_available():
        ref = O.Reference()
        return (lambda I, L, g, p, threads=1: ref.featurize(I, L, g, p, threads=threads)), \
            max(1, ref.max_threads())
    ora = O.Oracle()
    return (lambda I, L, g, p, threads=1: ora.featurize(I, L, g, p)), 1


def _compare(ctx, I, L, groups, profile):
    featurize, threads = _checker()
    gp = fx.resolve_profile(profile)
    cols = fx.feature_columns(groups, gp)
    gl, gv = ctx.featurize(I, L, groups, gp)
    rl, rv = featurize(I, L, groups, O.make_params(profile), threads)
    assert_parity(cols, gl, gv, rl, rv, I, L)
    return gl


def test_c2_bench_image(ctx):
    """bench.py's timed image itself (configs[1])."""
    import bench
    I, L, _ = bench.workload(0)
    gl = _compare(ctx, I, L, bench.GROUPS, bench.PROFILE)
    assert len(gl) == bench.ROI_COUNT


def test_c3_glcm_ibsi(ctx):
    L, _ = synth.packed_blob_mask_grid(4096, 400, 10000, 1)
    I = synth.uniform_u16(L.shape, 0)
    gl = _compare(ctx, I, L, ["glcm"], "ibsi-like")
    assert len(gl) == 10000


def test_c4_full_launch_set_all_groups(ctx):
    """512 tiles of 512^2 (one full launch set of table slots), ~100 ROIs each,
    every group: the batch path against the reference tile by tile."""
    n = 512
    tiles = []
    for s in range(n):
        L, _ = synth.packed_blob_mask_grid(512, 1000, 100, s % 64)
        tiles.append((synth.uniform_u16(L.shape, 1000 + s), L))
    p = fx.resolve_profile("default")
    cols = fx.feature_columns(ALL, p)
    res = ctx.featurize_batch(tiles, ALL, p)
    featurize, threads = _checker()
    op = O.make_params("default")
    with ThreadPoolExecutor(max(1, min(threads, os.cpu_count() or 1))) as ex:
        refs = list(ex.map(lambda t: featurize(t[0], t[1], ALL, op, 1), tiles))
    for (I, L), (gl, gv), (rl, rv) in zip(tiles, res, refs):
        assert_parity(cols, gl, gv, rl, rv, I, L)
    assert sum(len(r[0]) for r in res) >= 100 * n * 0.99


def test_c5_large_rois(ctx):
    """16384^2 slide of ~2e5-px blobs (all on the large-ROI CTA path), rolled so
    that blobs straddle the 8192-row band seam and the top/bottom ones wrap into
    two-component ROIs."""
    L, _ = synth.packed_blob_mask_grid(16384, 200000, 576, 1)
    L = np.roll(L, 340, axis=0)
    I = synth.uniform_u16(L.shape, 5)
    gl = _compare(ctx, I, L, ["intensity", "moments", "glcm"], "default")
    assert len(gl) == 576
