"""Pin the C restatement (oracle/fx_oracle.c) to the compiled reference
(oracle/_ref/libfxref.so, built from /root/reference/proj/src).

The restatement keeps the reference's fp operation order, so the two agree bit
for bit on every column; these tests assert exactly that on the synthetic
configs and on the adversarial masks.  CPU only.
"""
import numpy as np
import pytest

import inputs
from oracle import make_params

GROUPS = ["intensity", "shape", "moments", "glcm", "glrlm", "glszm", "ngtdm"]


def _blob(reference, size, roi_size, count, seed):
    return reference.blob_mask_grid(size, roi_size, count, seed)


@pytest.mark.parametrize("profile", ["default", "performance", "ibsi-like"])
def test_c1_shaped_bitwise(oracle, reference, profile):
    L = _blob(reference, 512, 300, 100, 7)
    I = inputs.uniform(L.shape, 0)
    p = make_params(profile)
    ol, ov = oracle.featurize(I, L, GROUPS, p)
    rl, rv = reference.featurize(I, L, GROUPS, p, threads=1)
    assert np.array_equal(ol, rl)
    assert np.array_equal(ov, rv)


@pytest.mark.parametrize("name", sorted(inputs.adversarial_masks()))
def test_adversarial_bitwise(oracle, reference, name):
    L = inputs.adversarial_masks()[name]
    for I in (inputs.uniform(L.shape, 1), np.zeros(L.shape, np.uint16),
              np.full(L.shape, 65535, np.uint16)):
        for profile in ("default", "performance"):
            p = make_params(profile)
            ol, ov = oracle.featurize(I, L, GROUPS, p)
            rl, rv = reference.featurize(I, L, GROUPS, p, threads=1)
            assert np.array_equal(ol, rl) and np.array_equal(ov, rv)


def test_star_and_random_labels_bitwise(oracle, reference):
    L = _blob(reference, 256, 220, 25, 5)
    I = reference.siemens_star(256)
    for over in ({}, dict(histogram_bins=7), dict(offset=2, ng=5), dict(angles=(135, 45))):
        p = make_params("default", **over)
        ol, ov = oracle.featurize(I, L, GROUPS, p)
        rl, rv = reference.featurize(I, L, GROUPS, p, threads=1)
        assert np.array_equal(ov, rv), over
    L = inputs.random_labels((40, 53), 7, seed=3)
    I = inputs.uniform(L.shape, 3)
    p = make_params("default")
    assert np.array_equal(oracle.featurize(I, L, GROUPS, p)[1],
                          reference.featurize(I, L, GROUPS, p, threads=1)[1])


def test_label_scan(oracle, reference):
    L = inputs.random_blobs((97, 131), 60, seed=2, label_values=np.array([1, 65535, 300, 4]))
    a = oracle.roi_table(L)
    b = reference.roi_table(np.zeros_like(L), L, rows_per_tile=7)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_contour_trace_identical(oracle, reference):
    rng = np.random.default_rng(0)
    for trial in range(300):
        h, w = rng.integers(3, 13, size=2)
        m = rng.random((h, w)) < rng.uniform(0.3, 0.9)
        ys, xs = np.nonzero(m)
        if len(xs) == 0:
            continue
        a = oracle.trace_contour(xs, ys)
        b = reference.trace_contour(xs, ys)
        assert np.array_equal(a, b)


def test_glcm_counts_match_reference_p(oracle, reference):
    rng = np.random.default_rng(1)
    for trial in range(40):
        h, w = rng.integers(2, 15, size=2)
        m = rng.random((h, w)) < 0.8
        m[0, 0] = True
        ys, xs = np.nonzero(m)
        vs = rng.integers(0, 900, len(xs)).astype(np.uint16)
        ng = int(rng.integers(2, 9))
        for ang in (0, 45, 90, 135):
            sym = bool(trial % 2)
            cnt, pairs = oracle.glcm_counts(xs, ys, vs, ng, 1, ang, sym)
            P, rp = reference.glcm(xs, ys, vs, ng, 1, ang, sym)
            assert pairs == rp
            if pairs:
                total = 2.0 * pairs if sym else float(pairs)
                assert np.array_equal(cnt / total, P)


def test_edge_definition_b_equals_trace(oracle):
    """trace_contour's visited set == pixels of the largest
    8-connected component K with a 4-neighbour in the 4-connected exterior of K
    (or on the bbox border).  The device edge kernel implements definition B."""
    from scipy import ndimage
    rng = np.random.default_rng(5)
    for trial in range(400):
        h, w = rng.integers(3, 16, size=2)
        m = rng.random((h, w)) < rng.uniform(0.3, 0.9)
        ys, xs = np.nonzero(m)
        if len(xs) == 0:
            continue
        y0, x0 = ys.min(), xs.min()
        sub = np.zeros((ys.max() - y0 + 1, xs.max() - x0 + 1), bool)
        sub[ys - y0, xs - x0] = True
        lab, n = ndimage.label(sub, structure=np.ones((3, 3)))
        sizes = np.bincount(lab.ravel())[1:]
        best = 1 + int(np.argmax(sizes))  # first max in label order == row-major first
        K = lab == best
        pad = np.pad(~K, 1, constant_values=True)
        elab, _ = ndimage.label(pad)
        E = elab == elab[0, 0]
        nb = E[:-2, 1:-1] | E[2:, 1:-1] | E[1:-1, :-2] | E[1:-1, 2:]
        edge = K & nb
        got = {(int(x + x0), int(y + y0)) for y, x in zip(*np.nonzero(edge))}
        pts = oracle.trace_contour(xs, ys)
        assert got == set(map(tuple, pts.tolist()))
