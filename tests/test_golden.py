"""Golden vectors of the reference's own unit tests, re-expressed (their doctest
suites do not build here: proj/vendor is absent), plus the committed reference
fixtures in tests/golden/ (made by tests/golden/make_golden.py from oracle/_ref).

CPU tests check the oracle; the gpu-marked tests check the device path against
the same numbers.  Sources (paths relative to /root/reference/proj):
  tests/test_intensity.cpp:29-79, tests/test_shape.cpp:32-140,
  tests/test_texture.cpp:45-126, tests/test_roistore.cpp:34-64,138-154,
  tests/test_engine.cpp:60-75,203-213.
"""
import glob
import os

import numpy as np
import pytest

from oracle import make_params
from parity import assert_parity

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = sorted(glob.glob(os.path.join(HERE, "golden", "*.npz")))
I_COLS = ["mean", "median", "mode", "min", "max", "range", "variance", "variance_biased", "std",
          "std_biased", "mad", "median_ad", "rmad", "iqr", "p1", "p10", "p25", "p75", "p90", "p99",
          "skewness", "kurtosis", "excess_kurtosis", "hyperskewness", "hyperflatness", "energy",
          "rms", "entropy", "uniformity", "qcod", "cov", "integrated_intensity", "edge_mean",
          "edge_min", "edge_max", "edge_std", "edge_integrated", "weighted_centroid_x",
          "weighted_centroid_y"]
G_COLS = ["asm", "acor", "cluprom", "clushade", "clutend", "contrast", "corr", "difave",
          "difentro", "difvar", "dis", "energy", "entropy", "hom1", "hom2", "id", "idn", "idm",
          "idmn", "infomeas1", "infomeas2", "iv", "jave", "je", "jmax", "jvar", "sumave",
          "sument", "sumvar"]


S_COLS = ["area", "perimeter", "bbox_x", "bbox_y", "bbox_w", "bbox_h", "centroid_x", "centroid_y",
          "circularity", "extent", "aspect_ratio", "convex_area", "solidity",
          "equivalent_diameter", "major_axis_len", "minor_axis_len", "eccentricity", "elongation",
          "orientation", "euler_number", "feret_max", "feret_min"] + [
          f"extrema_{c}_{a}" for c in ("topleft", "topright", "righttop", "rightbottom",
                                       "bottomright", "bottomleft", "leftbottom", "lefttop")
          for a in ("x", "y")]


def shape(fn, xs, ys):
    xs, ys = np.asarray(xs), np.asarray(ys)
    return dict(zip(S_COLS, fn(xs, ys, np.ones(len(xs), np.uint16), ["shape"],
                               make_params("default"))))


def run_shape_known_answers(fn):                                 # test_shape.cpp:32-120
    ys, xs = np.mgrid[3:13, 5:15]
    f = shape(fn, xs.ravel(), ys.ravel())                        # 10x10 solid square
    assert f["area"] == 100 and f["bbox_w"] == 10 and f["bbox_h"] == 10
    assert f["extent"] == pytest.approx(1) and f["euler_number"] == 1
    assert f["feret_max"] == pytest.approx(9 * np.sqrt(2)) and f["feret_min"] == pytest.approx(9)
    assert f["solidity"] == pytest.approx(1) and f["convex_area"] == pytest.approx(100)
    assert f["aspect_ratio"] == pytest.approx(1)
    ys, xs = np.nonzero(np.array([[1, 1, 1], [1, 0, 1], [1, 1, 1]]))
    assert shape(fn, xs, ys)["euler_number"] == 0                # one hole
    xs = np.arange(10)
    f = shape(fn, xs, np.full(10, 5))                            # 1x10 line
    mu20 = np.sum((xs - xs.mean()) ** 2) / 10 + 1 / 12
    mu02 = 1 / 12
    assert f["major_axis_len"] == pytest.approx(4 * np.sqrt(mu20), rel=1e-12)
    assert f["minor_axis_len"] == pytest.approx(4 * np.sqrt(mu02), rel=1e-12)
    assert f["eccentricity"] == pytest.approx(np.sqrt(1 - mu02 / mu20), rel=1e-12)
    assert f["orientation"] == pytest.approx(0) and f["minor_axis_len"] > 0
    f = shape(fn, [3], [4])                                      # single pixel
    assert f["area"] == 1 and f["perimeter"] == pytest.approx(4)
    assert f["circularity"] == pytest.approx(1) and f["convex_area"] == 0
    assert f["solidity"] == 0 and f["feret_max"] == 0
    f = shape(fn, [0, 1, 2], [0, 0, 0])                          # collinear cloud
    assert f["convex_area"] == 0 and f["solidity"] == 0
    assert f["feret_max"] == pytest.approx(2) and f["feret_min"] == 0


def line(values):
    v = np.asarray(values)
    return np.arange(len(v)), np.zeros(len(v)), v


def intensity(fn, xs, ys, vs, bins=256):
    p = make_params("default", histogram_bins=bins)
    return dict(zip(I_COLS, fn(xs, ys, vs, ["intensity"], p)))


def glcm_feats(fn, grid, ng, angle=0, symmetric=True):
    g = np.asarray(grid)
    ys, xs = np.nonzero(g >= 0)
    vs = g[ys, xs]
    p = make_params("default", ng=ng, angles=(angle,), symmetric=symmetric)
    out = fn(xs, ys, vs, ["glcm"], p)
    return {s: out[i * 2] for i, s in enumerate(G_COLS)}


def moments(fn, xs, ys, vs):
    p = make_params("default")
    out = fn(xs, ys, vs, ["moments"], p)
    names = []
    for pre in ("", "w"):
        names += [f"{pre}m{a}{b}" for a in range(4) for b in range(4)]
        names += [f"{pre}mu{a}{b}" for a in range(4) for b in range(4)]
        names += [f"{pre}eta{a}{b}" for a in range(4) for b in range(4) if a + b >= 2]
        names += [f"{pre}hu{k}" for k in range(1, 8)]
    return dict(zip(names, out))


def run_known_answers(fn):
    f = intensity(fn, *line([5, 5, 5, 5]))                     # test_intensity.cpp:29-41
    assert f["mean"] == 5 and f["variance"] == 0 and f["std"] == 0 and f["entropy"] == 0
    assert f["uniformity"] == pytest.approx(1) and f["energy"] == 100 and f["range"] == 0
    assert f["skewness"] == 0 and f["kurtosis"] == 0 and f["mode"] == 5
    f = intensity(fn, *line([0, 1, 2, 3]))                     # :43-52
    assert f["mean"] == 1.5 and f["variance_biased"] == pytest.approx(1.25)
    assert f["median"] == 1.5 and f["p25"] == 0.75 and f["p75"] == 2.25 and f["iqr"] == 1.5
    assert f["energy"] == 14
    f = intensity(fn, *line([2, 4]), bins=2)                   # :54-58
    assert f["entropy"] == pytest.approx(1.0) and f["uniformity"] == pytest.approx(0.5)
    f = intensity(fn, [3], [4], [9])                            # :60-79 weighted centroid
    assert (f["weighted_centroid_x"], f["weighted_centroid_y"]) == (3, 4)
    f = intensity(fn, [0, 2], [0, 0], [1, 3])
    assert (f["weighted_centroid_x"], f["weighted_centroid_y"]) == (1.5, 0)
    f = intensity(fn, [0, 2], [0, 0], [0, 0])                   # zero mass -> 0 (:205-213)
    assert (f["weighted_centroid_x"], f["weighted_centroid_y"]) == (0, 0)
    m = moments(fn, [3], [4], [5])                              # test_shape.cpp:124-133
    assert m["m00"] == 1 and all(m[f"mu{a}{b}"] == pytest.approx(0, abs=1e-15)
                                 for a in range(4) for b in range(4) if a + b >= 1)
    m = moments(fn, [0, 2], [0, 0], [1, 1])                     # :135-140
    assert m["mu20"] == pytest.approx(2) and m["mu02"] == 0 and m["hu1"] == pytest.approx(0.5)
    m = moments(fn, [0, 1], [0, 0], [0, 0])                     # zero weighted mass -> zeros
    assert all(v == 0 for k, v in m.items() if k.startswith("w"))
    g = glcm_feats(fn, [[5, 5, 5]] * 3, ng=4)                   # test_texture.cpp:98-107
    assert g["asm"] == pytest.approx(1) and g["contrast"] == 0 and g["entropy"] == 0
    g = glcm_feats(fn, [[10, 200], [200, 10]], ng=2)            # :109-117
    assert g["contrast"] == pytest.approx(1) and g["corr"] == pytest.approx(-1)
    assert g["idm"] == pytest.approx(0.5)
    g = glcm_feats(fn, [[77]], ng=4)                            # :119-126 one pixel
    assert all(v == 0 for v in g.values())


def test_known_answers_oracle(oracle):
    run_known_answers(oracle.roi_features)
    run_shape_known_answers(oracle.roi_features)


@pytest.mark.gpu
def test_known_answers_device(ctx):
    import paper_2603_12016_b200 as fx

    def fn(xs, ys, vs, groups, p):
        fp = fx.TextureParams()
        for k in ("ng", "offset", "n_angles", "symmetric", "histogram_bins"):
            setattr(fp, k, getattr(p, k))
        for i in range(8):
            fp.angles[i] = p.angles[i]
        return ctx.roi_features(xs, ys, vs, groups, fp)
    run_known_answers(fn)
    run_shape_known_answers(fn)


def test_label_scan_known_answer(oracle):                      # test_roistore.cpp:34-64
    labels, counts, bbox = oracle.roi_table(np.array([[0, 1], [1, 2]], np.uint16))
    assert labels.tolist() == [1, 2] and counts.tolist() == [2, 1]
    assert bbox.tolist() == [[0, 0, 1, 1], [1, 1, 1, 1]]
    assert len(oracle.roi_table(np.zeros((3, 3), np.uint16))[0]) == 0


def test_contour_known_answers(oracle):                        # test_roistore.cpp:138-154
    assert oracle.trace_contour([3], [4]).tolist() == [[3, 4]]
    ys, xs = np.mgrid[0:3, 0:3]
    pts = set(map(tuple, oracle.trace_contour(xs.ravel(), ys.ravel()).tolist()))
    assert len(pts) == 8 and (1, 1) not in pts


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p)[:-4] for p in GOLDEN])
def test_golden_fixture_oracle(oracle, path):
    d = np.load(path)
    for prof in ("default", "performance", "ibsi-like"):
        ol, ov = oracle.featurize(d["intensity"], d["labels"], ["intensity", "moments", "glcm"],
                                  make_params(prof))
        assert np.array_equal(ol, d[f"{prof}_labels"])
        assert np.array_equal(ov, d[f"{prof}_values"])


@pytest.mark.gpu
@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p)[:-4] for p in GOLDEN])
def test_golden_fixture_device(ctx, path):
    import paper_2603_12016_b200 as fx
    d = np.load(path)
    for prof in ("default", "performance", "ibsi-like"):
        p = fx.resolve_profile(prof)
        cols = fx.feature_columns(["intensity", "moments", "glcm"], p)
        assert cols == d[f"{prof}_columns"].tolist()
        gl, gv = ctx.featurize(d["intensity"], d["labels"], ["intensity", "moments", "glcm"], p)
        assert_parity(cols, gl, gv, d[f"{prof}_labels"], d[f"{prof}_values"], d["intensity"],
                      d["labels"])
