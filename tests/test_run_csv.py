"""Drop-in check at the file level: featurex::run of this repo (fx.run -> the C++
engine's batched pipeline on the GPU) against the reference's own featurex::run
(oracle/_ref, engine.cpp:283-350) on the same PGM directories.

Same summary (images, ROIs, rows, failed pairs), same header and row keys in the
same order, and every value within the parity rules of tests/parity.py (the
CSV's %.10g rounding, <= 5e-11 relative per side, sits inside them; bit-exact
columns compare equal as text because equal doubles print equally).
"""
import csv

import numpy as np
import pytest

import inputs
from parity import assert_parity

import paper_2603_12016_b200 as fx
from tools import synth

pytestmark = pytest.mark.gpu


def _pairs():
    rng = np.random.default_rng(5)
    out = {}
    L = synth.blob_mask_grid(256, 200, 40, 2)
    out["a_blobs.pgm"] = (synth.uniform_u16(L.shape, 3), L, 65535, 65535)
    S = synth.siemens_star(128)
    Ls = synth.blob_mask_grid(128, 200, 9, 4)
    out["b_star.pgm"] = (S, Ls, 65535, 65535)
    Lt, _ = synth.packed_blob_mask_grid(192, 250, 30, 6)
    out["c_tertiary.pgm"] = (inputs.per_roi_levels(Lt, 7), Lt, 65535, 255)
    Lr = inputs.random_blobs((90, 140), 25, seed=8)
    out["d_random.pgm"] = (rng.integers(0, 4096, Lr.shape).astype(np.uint16), Lr, 4095, 255)
    L8 = synth.blob_mask_grid(64, 80, 6, 9)
    out["e_8bit.pgm"] = (rng.integers(0, 256, L8.shape).astype(np.uint16), L8, 255, 255)
    Lw = np.zeros((300, 280), np.uint16)
    Lw[20:260, 30:250] = 3  # a window wider and taller than 64 (large-ROI path)
    Lw[100:140, 100:160] = 0
    out["f_large.pgm"] = (rng.integers(0, 65536, Lw.shape).astype(np.uint16), Lw, 65535, 255)
    out["g_empty.pgm"] = (rng.integers(0, 65536, (16, 16)).astype(np.uint16),
                          np.zeros((16, 16), np.uint16), 65535, 255)
    return out


def _read(path):
    with open(path) as f:
        r = csv.reader(f)
        head = next(r)
        rows = list(r)
    return head, rows


@pytest.mark.parametrize("groups", [["*ALL*"], ["intensity", "moments", "glcm"]])
def test_run_matches_reference_run(reference, tmp_path, groups):
    pairs = _pairs()
    for sub in ("int", "seg"):
        (tmp_path / sub).mkdir()
    for name, (I, L, mi, ml) in pairs.items():
        fx.write_pgm(tmp_path / "int" / name, I, mi)
        fx.write_pgm(tmp_path / "seg" / name, L, ml)
    (tmp_path / "int" / "h_corrupt.pgm").write_bytes(b"P5\n4 4\n255\nX")
    fx.write_pgm(tmp_path / "seg" / "h_corrupt.pgm", np.ones((4, 4), np.uint16), 255)
    fx.write_pgm(tmp_path / "seg" / "i_orphan.pgm", np.ones((4, 4), np.uint16), 255)

    ours = fx.run(tmp_path / "int", tmp_path / "seg", groups, output_path=tmp_path / "ours.csv")
    ref = reference.run(tmp_path / "int", tmp_path / "seg", groups, threads=reference.max_threads(),
                        output_path=tmp_path / "ref.csv")
    assert (ours.images, ours.rois, ours.rows, ours.failed_pairs) == \
        (ref.images, ref.rois, ref.rows, ref.failed_pairs)
    assert ours.failed_pairs == 2 and ours.images == len(pairs)

    h1, r1 = _read(tmp_path / "ours.csv")
    h2, r2 = _read(tmp_path / "ref.csv")
    assert h1 == h2
    assert [row[:3] for row in r1] == [row[:3] for row in r2]
    cols = h1[3:]
    for name, (I, L, _, _) in pairs.items():
        mine = [row for row in r1 if row[0] == name]
        theirs = [row for row in r2 if row[0] == name]
        if not theirs:
            continue
        gl = np.array([int(row[2]) for row in mine])
        gv = np.array([[float(x) for x in row[3:]] for row in mine])
        rv = np.array([[float(x) for x in row[3:]] for row in theirs])
        assert_parity(cols, gl, gv, gl, rv, I, L)
