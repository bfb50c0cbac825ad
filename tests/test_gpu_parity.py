"""GPU parity: the sm_100a path through the C ABI vs the oracle.

The oracle is the C restatement (oracle/fx_oracle.c), itself pinned bit-for-bit
against the compiled reference in test_oracle_pin.py; where the compiled
reference (oracle/_ref) is present it is checked directly as well.
"""
import numpy as np
import pytest

import inputs
from parity import assert_parity

import paper_2603_12016_b200 as fx
from tools import synth
from oracle import make_params as oparams

pytestmark = pytest.mark.gpu

GROUPS = ["intensity", "shape", "moments", "glcm", "glrlm", "glszm", "ngtdm"]


def both_params(profile="default", **over):
    return fx.make_params(profile, **over), oparams(profile, **over)


def check(ctx, oracle, I, L, groups, profile="default", **over):
    gp, op = both_params(profile, **over)
    cols = fx.feature_columns(groups, gp)
    gl, gv = ctx.featurize(I, L, groups, gp)
    ol, ov = oracle.featurize(I, L, groups, op)
    assert_parity(cols, gl, gv, ol, ov, I, L)
    return gl, gv


@pytest.mark.parametrize("profile", ["default", "performance", "ibsi-like"])
def test_c1_blob_grid_all_groups(ctx, oracle, profile):
    L = synth.blob_mask_grid(1024, 421, 500, 1)
    I = synth.uniform_u16(L.shape, 0)
    gl, _ = check(ctx, oracle, I, L, GROUPS, profile)
    assert len(gl) == 500


@pytest.mark.parametrize("groups", [["intensity"], ["moments"], ["glcm"], ["intensity", "glcm"]])
def test_group_subsets(ctx, oracle, groups):
    L = synth.blob_mask_grid(512, 300, 100, 7)
    I = synth.siemens_star(512)
    check(ctx, oracle, I, L, groups)


def test_tertiary_intensities(ctx, oracle):
    L, _ = synth.packed_blob_mask_grid(768, 600, 250, 3)
    I = inputs.per_roi_levels(L, 5)
    check(ctx, oracle, I, L, GROUPS)


@pytest.mark.parametrize("name", sorted(inputs.adversarial_masks()))
def test_adversarial_masks(ctx, oracle, name):
    L = inputs.adversarial_masks()[name]
    for seed, I in enumerate([inputs.uniform(L.shape, 1), np.full(L.shape, 77, np.uint16),
                              np.zeros(L.shape, np.uint16),
                              np.full(L.shape, 65535, np.uint16)]):
        check(ctx, oracle, I, L, GROUPS)
        check(ctx, oracle, I, L, GROUPS, "performance")


def _value_distributions(shape):
    """Intensity laws that drive each branch of the warp value sort: narrow range
    (buckets are single values), 12-bit (in-bucket ranking), two modes and a narrow
    body with rare extremes (crowded buckets, radix fallback)."""
    rng = np.random.default_rng(11)
    narrow = rng.integers(1000, 1300, shape).astype(np.uint16)
    twelve = rng.integers(0, 4096, shape).astype(np.uint16)
    bimodal = np.where(rng.random(shape) < 0.5, 0, 65535).astype(np.uint16)
    outliers = rng.integers(500, 520, shape).astype(np.uint16)
    outliers[rng.random(shape) < 0.01] = 65535
    return {"narrow": narrow, "twelve_bit": twelve, "bimodal": bimodal, "outliers": outliers}


@pytest.mark.parametrize("law", ["narrow", "twelve_bit", "bimodal", "outliers"])
def test_value_sort_branches(ctx, oracle, law):
    L, _ = synth.packed_blob_mask_grid(1024, 700, 300, 5)
    I = _value_distributions(L.shape)[law]
    check(ctx, oracle, I, L, ["intensity", "moments"])
    check(ctx, oracle, I, L, GROUPS)


@pytest.mark.parametrize("seed", range(6))
def test_random_blobs(ctx, oracle, seed):
    L = inputs.random_blobs((96, 130), 40, seed=seed)
    I = inputs.uniform(L.shape, seed)
    check(ctx, oracle, I, L, GROUPS)


@pytest.mark.parametrize("shape,n", [((20, 20), 6), ((64, 64), 9), ((150, 97), 5)])
def test_random_label_masks_large_windows(ctx, oracle, shape, n):
    """labels scattered over the whole image: windows exceed the S tile -> L path"""
    L = inputs.random_labels(shape, n, seed=11)
    I = inputs.uniform(shape, 2)
    check(ctx, oracle, I, L, GROUPS)


def test_large_roi_l_path(ctx, oracle):
    yy, xx = np.mgrid[0:300, 0:260]
    L = np.zeros((300, 260), np.uint16)
    L[(xx - 130) ** 2 / 110.0 ** 2 + (yy - 150) ** 2 / 140.0 ** 2 <= 1] = 3
    L[20:40, 10:200] = 9
    I = inputs.uniform(L.shape, 9)
    check(ctx, oracle, I, L, GROUPS)


def test_odd_width_no_tma(ctx, oracle):
    L = synth.blob_mask_grid(331, 200, 40, 2)[:, :329].copy()
    I = inputs.uniform(L.shape, 4)
    check(ctx, oracle, I, L, GROUPS)


def test_histogram_bins_and_offsets(ctx, oracle):
    L = synth.blob_mask_grid(256, 220, 25, 5)
    I = inputs.uniform(L.shape, 6)
    for over in [dict(histogram_bins=2), dict(histogram_bins=1000), dict(offset=2),
                 dict(ng=2), dict(ng=7, symmetric=False, angles=(135, 0, 45)),
                 dict(angles=(90, 90))]:
        check(ctx, oracle, I, L, GROUPS, **over)


def test_empty_mask(ctx):
    L = np.zeros((64, 64), np.uint16)
    I = inputs.uniform(L.shape, 0)
    gl, gv = ctx.featurize(I, L, GROUPS)
    assert len(gl) == 0 and gv.shape[0] == 0


def test_label_scan_bit_exact(ctx, oracle):
    for L in [synth.blob_mask_grid(1024, 421, 500, 1), inputs.random_labels((77, 1003), 300, 3),
              inputs.random_blobs((257, 513), 200, seed=4,
                                  label_values=np.array([1, 2, 65535, 40000, 17]))]:
        gl, gc, gb = ctx.roi_table(np.zeros_like(L), L)
        ol, oc, ob = oracle.roi_table(L)
        assert np.array_equal(gl, ol) and np.array_equal(gc, oc) and np.array_equal(gb, ob)


def test_label_scan_evicted_largest_label(ctx, oracle):
    """The largest label of a strip leaves a lane's 2-entry cache before the strip
    ends (three labels down one 8-px column): it must still raise the slot's max
    label, or compaction skips its 1024-label block, drops the ROI and leaves its
    table entry to leak into the next call."""
    for big in (1024, 40000, 65535):
        L = np.zeros((70, 40), np.uint16)
        L[0:3, 0:5] = big
        L[3:5, 0:8] = 1
        L[5:9, 0:8] = 2
        L[20:22, 9:20] = big - 1
        L[22, 9:20] = 3
        L[23, 9:20] = 4
        for _ in range(2):  # twice: a leaked entry would double the second count
            gl, gc, gb = ctx.roi_table(np.zeros_like(L), L)
            ol, oc, ob = oracle.roi_table(L)
            assert np.array_equal(gl, ol) and np.array_equal(gc, oc) and np.array_equal(gb, ob)
        check(ctx, oracle, inputs.uniform(L.shape, 1), L, GROUPS)


@pytest.mark.parametrize("rows", [32, 63, 64])
def test_two_components_touching_last_window_row(ctx, oracle, rows):
    """A two-component ROI whose window is `rows` tall, the components at the top and
    on the last row (found by the randomized sweep: a 64-row window lost its bottom
    Euler quads, took the one-component fast path and merged both edge sets)."""
    L = np.zeros((rows + 6, 60), np.uint16)
    L[3:3 + 12, 40:53] = 9                 # top component
    L[3 + rows - 8:3 + rows, 2:27] = 9     # bottom component, on the window's last row
    L[3 + rows - 1, 12:17] = 0             # a notch: two runs on that row
    L[3 + rows - 3, 5:9] = 0
    I = inputs.uniform(L.shape, 2)
    check(ctx, oracle, I, L, GROUPS)
    ys, xs = np.nonzero(L == 9)
    _, edge, _, _ = ctx.debug_roi(I, L, 9, fx.make_params("default"))
    assert set(map(tuple, edge.tolist())) == set(map(tuple, oracle.trace_contour(xs, ys).tolist()))


@pytest.mark.parametrize("hw", [(7, 5), (3, 30), (40, 60), (90, 20), (150, 150)])
def test_single_run_cell_entropy_is_zero(ctx, oracle, hw):
    """Constant-intensity rectangles: at 0 and 90 degrees every run falls in one
    (level, length) cell, so run entropy is exactly 0 in the reference; the device
    sums must cancel exactly too (a 1-ulp residue is an infinite relative error)."""
    h, w = hw
    L = np.zeros((h + 4, w + 4), np.uint16)
    L[2:2 + h, 2:2 + w] = 7
    I = np.full(L.shape, 1234, np.uint16)
    gl, gv = check(ctx, oracle, I, L, ["glrlm"], angles=(0, 90))
    cols = fx.feature_columns(["glrlm"], fx.make_params("default", angles=(0, 90)))
    for c in ("glrlm_re_0", "glrlm_re_90"):
        assert gv[0, cols.index(c)] == 0.0


def test_debug_histogram_edges_glcm_bit_exact(ctx, oracle):
    masks = inputs.adversarial_masks()
    masks["blobs"] = synth.blob_mask_grid(256, 220, 25, 5)
    p = fx.make_params("default", histogram_bins=16)
    for name, L in masks.items():
        I = inputs.uniform(L.shape, 3)
        for lab in np.unique(L[L > 0])[:6]:
            ys, xs = np.nonzero(L == lab)
            vs = I[ys, xs]
            hist, edge, glcm, pairs = ctx.debug_roi(I, L, int(lab), p)
            assert np.array_equal(hist, oracle.intensity_hist(vs, 16)), name
            pts = oracle.trace_contour(xs, ys)
            assert set(map(tuple, edge.tolist())) == set(map(tuple, pts.tolist())), (name, lab)
            for a, ang in enumerate(sorted(p.angles[: p.n_angles])):
                cnt, pc = oracle.glcm_counts(xs, ys, vs, p.ng, p.offset, ang, p.symmetric)
                assert pairs[a] == pc, (name, lab, ang)
                assert np.array_equal(glcm[a].astype(np.uint64), cnt), (name, lab, ang)


def test_per_roi_operator(ctx, oracle):
    rng = np.random.default_rng(3)
    for trial in range(10):
        L = inputs.random_blobs((40, 40), 3, seed=trial, label_values=np.array([1]))
        ys, xs = np.nonzero(L)
        if len(xs) == 0:
            continue
        xs = xs + 1000 * trial
        ys = ys + 37
        vs = rng.integers(0, 4000, len(xs)).astype(np.uint16)
        gp, op = both_params("default")
        g = ctx.roi_features(xs, ys, vs, GROUPS, gp)
        o = oracle.roi_features(xs, ys, vs, GROUPS, op)
        assert_parity(fx.feature_columns(GROUPS, gp), [1], g[None], [1], o[None])


def test_per_roi_operator_rejects_repeated_pixels(ctx):
    """A PixelCloud holds each pixel once; a repeated one is an argument error, not
    a silently different table (the rasterized cloud would count it once)."""
    xs = np.array([3, 4, 5, 4], np.uint32)
    ys = np.array([7, 7, 7, 7], np.uint32)
    vs = np.array([10, 20, 30, 40], np.uint16)
    with pytest.raises(fx.FxError) as e:
        ctx.roi_features(xs, ys, vs, GROUPS)
    assert e.value.kind == "ArgumentError" and "duplicate" in str(e.value)
    with pytest.raises(fx.FxError) as e:
        ctx.roi_features_batch([(xs[:3], ys[:3], vs[:3]), (xs, ys, vs)], GROUPS)
    assert e.value.kind == "ArgumentError" and "cloud 1" in str(e.value)
    ctx.roi_features(xs[:3], ys[:3], vs[:3], GROUPS)  # the context stays usable


def test_vs_compiled_reference(ctx, reference):
    L = synth.blob_mask_grid(512, 300, 100, 7)
    I = synth.uniform_u16(L.shape, 0)
    gp, op = both_params("default")
    cols = fx.feature_columns(GROUPS, gp)
    gl, gv = ctx.featurize(I, L, GROUPS, gp)
    rl, rv = reference.featurize(I, L, GROUPS, op)
    assert_parity(cols, gl, gv, rl, rv, I, L)


def _exact_central(xs, ys, w, p, q):
    from fractions import Fraction
    W = int(w.sum())
    cx = Fraction(int((w * xs).sum()), W)
    cy = Fraction(int((w * ys).sum()), W)
    return sum(Fraction(int(a)) * (Fraction(int(x)) - cx) ** p * (Fraction(int(y)) - cy) ** q
               for a, x, y in zip(w, xs, ys))


def test_moments_vs_exact_rational_truth(ctx):
    """The device's central moments are computed about integer anchors and are
    checked against exact rational arithmetic at 1e-12 of the natural scale
    (the reference itself misses 1e-9 on some of these, see parity.py)."""
    import os
    from parity import _moment_scales
    d = np.load(os.path.join(os.path.dirname(__file__), "golden", "blobs_star.npz"))
    cases = [(d["intensity"], d["labels"]),
             (inputs.uniform((96, 130), 3), inputs.random_blobs((96, 130), 30, seed=3))]
    for I, L in cases:
        p = fx.resolve_profile("default")
        cols = fx.feature_columns(["moments"], p)
        gl, gv = ctx.featurize(I, L, ["moments"], p)
        nat = _moment_scales(I, L, gl, reference_frame=False)
        for k, lab in enumerate(gl[:8]):
            ys, xs = np.nonzero(L == lab)
            for g, pre in enumerate(("", "w")):
                w = np.ones(len(xs), np.int64) if g == 0 else I[ys, xs].astype(np.int64)
                if w.sum() == 0:
                    continue
                for (a, b) in ((2, 0), (1, 1), (3, 0), (2, 1), (3, 3), (2, 3)):
                    ex = float(_exact_central(xs, ys, w, a, b))
                    got = gv[k, cols.index(f"moments_{pre}mu{a}{b}")]
                    assert abs(got - ex) <= 1e-12 * (abs(ex) + nat[k, g, a, b]), (lab, pre, a, b)
                raw = float(sum(int(c) * int(x) ** 3 * int(y) ** 3 for c, x, y in zip(w, xs, ys)))
                assert abs(gv[k, cols.index(f"moments_{pre}m33")] - raw) <= 1e-14 * abs(raw)


# ---- large-ROI path (k_roi_b: one CTA per ROI) ------------------------------

def _large_masks():
    """Windows > 64: big disc/ring with holes, two equal-size components of one
    label (row-major tie-break), a spiral-ish comb, a thin diagonal, sparse pixels."""
    yy, xx = np.mgrid[0:300, 0:280]
    L = np.zeros((300, 280), np.uint16)
    r2 = (xx - 140) ** 2 + (yy - 150) ** 2
    L[(r2 <= 120 ** 2) & (r2 >= 30 ** 2)] = 5                 # ring: one big hole
    L[(r2 <= 12 ** 2)] = 5                                     # island inside the hole
    L[((xx - 140) ** 2 + (yy - 150) ** 2 <= 60 ** 2) & ((xx + yy) % 17 == 0)] = 0  # slits
    L[5:25, 5:80] = 7
    L[270:290, 190:265] = 7                                    # equal-size twin
    for k in range(0, 260, 8):
        L[k:k + 4, 270:278] = 9                                # comb teeth
    L[0:300:1, 279] = 9
    for d in range(0, 250):
        L[40 + d // 2, 10 + d // 3] = 11                        # thin diagonal
    rng = np.random.default_rng(4)
    L[rng.integers(0, 300, 400), rng.integers(0, 280, 400)] = 13  # scattered pixels
    return L


@pytest.mark.parametrize("profile", ["default", "performance", "ibsi-like"])
@pytest.mark.parametrize("fill", ["uniform", "levels", "constant"])
def test_large_rois_cta_path(ctx, oracle, profile, fill):
    L = _large_masks()
    I = {"uniform": inputs.uniform(L.shape, 6), "levels": inputs.per_roi_levels(L, 2),
         "constant": np.full(L.shape, 321, np.uint16)}[fill]
    check(ctx, oracle, I, L, GROUPS, profile)


def test_large_rois_cta_debug_bit_exact(ctx, oracle):
    """Histogram counts, edge pixel set and GLCM counts of large ROIs, ng 64 and 256."""
    L = _large_masks()
    I = inputs.uniform(L.shape, 8)
    for profile, bins in [("default", 16), ("ibsi-like", 300)]:
        p = fx.make_params(profile, histogram_bins=bins)
        for lab in [5, 7, 9, 11, 13]:
            ys, xs = np.nonzero(L == lab)
            vs = I[ys, xs]
            hist, edge, glcm, pairs = ctx.debug_roi(I, L, int(lab), p)
            assert np.array_equal(hist, oracle.intensity_hist(vs, bins)), lab
            pts = oracle.trace_contour(xs, ys)
            assert set(map(tuple, edge.tolist())) == set(map(tuple, pts.tolist())), lab
            for a, ang in enumerate(sorted(p.angles[: p.n_angles])):
                cnt, pc = oracle.glcm_counts(xs, ys, vs, p.ng, p.offset, ang, p.symmetric)
                assert pairs[a] == pc, (lab, ang)
                assert np.array_equal(glcm[a].astype(np.uint64), cnt), (lab, ang)


def test_large_rois_deterministic(ctx):
    L = _large_masks()
    I = inputs.uniform(L.shape, 1)
    a = ctx.featurize(I, L, GROUPS)
    for _ in range(4):
        b = ctx.featurize(I, L, GROUPS)
        assert np.array_equal(a[1], b[1])


def test_roi_features_batch_equals_per_cloud(ctx):
    """fx_roi_features_batch (one device pass for many clouds) == one
    fx_roi_features call per cloud, bit for bit: small, empty, single-pixel and
    large-window (L path) clouds, several launch sets."""
    rng = np.random.default_rng(9)
    clouds = []
    for k in range(700):
        r = 2 + k % 11
        yy, xx = np.nonzero(np.hypot(*np.mgrid[-r:r + 1, -r:r + 1]) <= r)
        keep = rng.random(len(xx)) < 0.85
        xs = (xx[keep] + 50 + 3 * k).astype(np.uint32)
        ys = (yy[keep] + 20 + k).astype(np.uint32)
        clouds.append((xs, ys, rng.integers(0, 65536, len(xs)).astype(np.uint16)))
    clouds[5] = (np.zeros(0, np.uint32), np.zeros(0, np.uint32), np.zeros(0, np.uint16))
    clouds[6] = (np.array([7], np.uint32), np.array([3], np.uint32), np.array([5], np.uint16))
    yy, xx = np.nonzero(np.ones((90, 120), bool))
    clouds[7] = (xx.astype(np.uint32), yy.astype(np.uint32),
                 rng.integers(0, 4096, len(xx)).astype(np.uint16))
    for groups in (["intensity", "moments"], ["*ALL*"]):
        got = ctx.roi_features_batch(clouds, groups)
        for k in (0, 5, 6, 7, 123, 699):
            want = ctx.roi_features(*clouds[k], groups)
            assert np.array_equal(got[k], want, equal_nan=True), (groups, k)


def test_unstaged_in_warp_paths(oracle, monkeypatch):
    """The in-warp intensity statistics and moments (taken when the staging buffers
    for the serial passes overflow, e.g. on huge images; forced here with
    FXG_NO_STAGE=1) match the oracle like the staged serial passes."""
    monkeypatch.setenv("FXG_NO_STAGE", "1")
    c = fx.Context(0)
    try:
        for L, I in [(synth.blob_mask_grid(512, 300, 100, 7), None),
                     (inputs.random_blobs((96, 130), 40, seed=2), None)]:
            I = inputs.uniform(L.shape, 3) if I is None else I
            check(c, oracle, I, L, ["intensity", "moments"])
            check(c, oracle, I, L, GROUPS)
    finally:
        c.close()


@pytest.mark.parametrize("spread", [1, 3, 40])
def test_tied_values_small_rois(ctx, oracle, spread):
    """Heavy ties around the median (the median split of the median absolute
    deviation, intensity_features.cpp:96-101) on ROIs of 1..16 pixels of both
    parities, plus blob ROIs of a few hundred pixels over a handful of levels."""
    rng = np.random.default_rng(spread)
    L = np.zeros((96, 96), np.uint16)
    lab = 1
    for y in range(0, 96, 4):
        for x in range(0, 96, 4):
            keep = rng.random((4, 4)) < 0.45
            L[y:y + 4, x:x + 4][keep] = lab
            lab += 1
    I = rng.integers(1000, 1000 + spread, size=L.shape, dtype=np.uint16)
    check(ctx, oracle, I, L, ["intensity", "moments"])
    Lb = synth.blob_mask_grid(512, 300, 100, 5)
    Ib = rng.integers(7, 7 + spread, size=Lb.shape, dtype=np.uint16)
    check(ctx, oracle, Ib, Lb, ["intensity", "moments"])


# ---- texture groups with more than 256 grey levels (the wide kernel) ----------

TEXTURE = ["glcm", "glrlm", "glszm", "ngtdm"]


@pytest.mark.parametrize("over", [dict(ng=512), dict(ng=300, symmetric=False, angles=(135, 0, 45)),
                                  dict(ng=2000, angles=(90, 90)), dict(ng=257, offset=2),
                                  dict(ng=4096)])
def test_wide_grey_levels(ctx, oracle, over):
    """ng > 256 (the reference accepts any ng >= 2, its level grid is int16): every
    texture group against the oracle, with the other groups alongside."""
    L = inputs.random_blobs((120, 150), 30, seed=3, max_r=14)
    I = inputs.uniform(L.shape, 7)
    check(ctx, oracle, I, L, GROUPS, **over)
    check(ctx, oracle, I, L, TEXTURE, **over)


def test_wide_grey_levels_tiles_and_large_rois(ctx, oracle):
    """ng = 512 on blob tiles (S windows) and on windows beyond 64 x 64 (L windows)"""
    L, _ = synth.packed_blob_mask_grid(512, 1000, 100, 3)
    I = synth.uniform_u16(L.shape, 2)
    check(ctx, oracle, I, L, GROUPS, ng=512)
    yy, xx = np.mgrid[0:300, 0:260]
    L = np.zeros((300, 260), np.uint16)
    L[(xx - 130) ** 2 / 110.0 ** 2 + (yy - 150) ** 2 / 140.0 ** 2 <= 1] = 3
    L[20:40, 10:200] = 9
    I = inputs.per_roi_levels(L, 4, noise=900)
    check(ctx, oracle, I, L, TEXTURE, ng=1024)


def test_wide_grey_levels_int16_limit(ctx, oracle):
    """ng = 32768, the largest level count of the reference's int16 grid (run-length
    and zone groups: the oracle's GLCM / NGTDM are O(ng^2) there)"""
    L = inputs.random_blobs((60, 70), 12, seed=8, max_r=10)
    I = inputs.uniform(L.shape, 9)
    check(ctx, oracle, I, L, ["intensity", "glrlm", "glszm"], ng=32768)


def test_wide_grey_levels_above_int16_is_config_error(ctx):
    L = inputs.random_blobs((40, 40), 5, seed=1)
    I = inputs.uniform(L.shape, 1)
    with pytest.raises(fx.FxError) as e:
        ctx.featurize(I, L, ["glcm"], fx.make_params("default", ng=40000))
    assert e.value.kind == "ConfigError"
