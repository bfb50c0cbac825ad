"""Host packer of the packed host rows (csrc/fx_pack.cpp), on the CPU: every
region decodes back to the rasters it came from (labels everywhere, intensities
exactly at the labelled pixels), the per-tile indices are the counts before each
2048-pixel tile, and a block that does not fit reports 0 bytes (sent raw).  The
device unpack of the same regions is covered by tests/test_batch.py (GPU)."""
import ctypes as C

import numpy as np
import pytest

import inputs

TILE = 2048


def _lib():
    from paper_2603_12016_b200 import fxg
    L = fxg.lib()
    L.fx_debug_pack_rows.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_int, C.c_void_p,
                                     C.c_size_t, C.c_void_p, C.c_size_t, C.POINTER(C.c_size_t),
                                     C.POINTER(C.c_size_t)]
    return L


def _pack(L, I, lab_cap=None, int_cap=None):
    rows, w = L.shape
    pitch = L.strides[0] // 2
    tiles = (w + TILE - 1) // TILE
    idx = (4 * (rows * tiles + 1) + 15) // 16 * 16
    lab_cap = lab_cap if lab_cap is not None else idx + 4 * rows * w + 128
    int_cap = int_cap if int_cap is not None else idx + 2 * rows * w + 64
    lr = np.zeros(lab_cap, np.uint8)
    ir = np.zeros(int_cap, np.uint8)
    lb, ib = C.c_size_t(), C.c_size_t()
    rc = _lib().fx_debug_pack_rows(L.ctypes.data, I.ctypes.data, pitch, w, rows, lr.ctypes.data, lab_cap,
                                   ir.ctypes.data, int_cap, C.byref(lb), C.byref(ib))
    if rc == 1:  # FX_E_CONFIG: no AVX-512 VBMI2 on this host (packing off)
        pytest.skip("host packer unavailable")
    assert rc == 0
    return lr, ir, lb.value, ib.value, tiles, idx


def _decode(L, I, lr, ir, lb, ib, tiles, idx):
    rows, w = L.shape
    tseg = lr[:4 * (rows * tiles + 1)].view(np.uint32)
    seg = lr[idx:lb].view(np.uint32)
    assert len(seg) == tseg[-1]
    tpix = ir[:4 * (rows * tiles + 1)].view(np.uint32)
    pix = ir[idx:ib].view(np.uint16)
    assert len(pix) == tpix[-1]
    outL = np.zeros_like(L)
    for y in range(rows):
        s0, s1 = int(tseg[y * tiles]), int(tseg[(y + 1) * tiles])
        xs = (seg[s0:s1] & 0xffff).astype(np.int64)
        ls = (seg[s0:s1] >> 16).astype(np.uint16)
        assert xs[0] == 0 and np.all(np.diff(xs) > 0)
        ends = np.append(xs[1:], w)
        for x, e, lab in zip(xs, ends, ls):
            outL[y, x:e] = lab
        for t in range(tiles):  # segments before each tile start / labelled pixels before it
            assert tseg[y * tiles + t] == s0 + np.count_nonzero(xs < t * TILE)
            assert tpix[y * tiles + t] == tpix[y * tiles] + np.count_nonzero(L[y, :t * TILE])
    assert np.array_equal(outL, L)
    assert np.array_equal(pix, I[L != 0])


def _cases():
    rng = np.random.default_rng(2)
    yield "blobs", inputs.random_blobs((300, 700), 60, seed=1, max_r=30,
                                       label_values=np.array([1, 65535, 40000, 2]))
    yield "noise", rng.integers(0, 65536, (40, 100)).astype(np.uint16)
    yield "empty", np.zeros((17, 64), np.uint16)
    yield "full", np.full((9, 31), 7, np.uint16)
    yield "width1", rng.integers(0, 3, (50, 1)).astype(np.uint16)
    yield "three_tiles", inputs.random_labels((12, 4097), 30, seed=3, p_bg=0.5)
    edge = np.zeros((6, 4100), np.uint16)
    edge[:, 2047:2049] = 5  # a run across the tile boundary
    edge[:, 4096:] = 9      # labels in the last partial vector
    edge[3, 0] = 1
    yield "tile_edges", edge


@pytest.mark.parametrize("name,L", list(_cases()), ids=[n for n, _ in _cases()])
def test_pack_roundtrip(name, L):
    I = inputs.uniform(L.shape, 4)
    lr, ir, lb, ib, tiles, idx = _pack(L, I)
    assert lb > 0 and ib > 0
    _decode(L, I, lr, ir, lb, ib, tiles, idx)


def test_pack_pitched_rows():
    L = inputs.random_blobs((64, 200), 20, seed=5, max_r=12)
    I = inputs.uniform(L.shape, 5)
    Lp = np.zeros((64, 256), np.uint16)
    Ip = np.zeros((64, 256), np.uint16)
    Lp[:, :200], Ip[:, :200] = L, I
    Lp[:, 200:] = 77  # outside the width: never packed
    lr, ir, lb, ib, tiles, idx = _pack(Lp[:, :200], Ip[:, :200])
    _decode(L, I, lr, ir, lb, ib, tiles, idx)


def test_pack_capacity_reports_raw():
    rng = np.random.default_rng(9)
    L = rng.integers(1, 65536, (32, 128)).astype(np.uint16)  # a change at every pixel
    I = inputs.uniform(L.shape, 1)
    rows, w = L.shape
    idx = (4 * (rows + 1) + 15) // 16 * 16
    _, _, lb, ib, _, _ = _pack(L, I, lab_cap=idx + 128 + rows * w)  # room for rows*w/4 segments
    assert lb == 0 and ib == 0
    _, _, lb, ib, _, _ = _pack(L, I, int_cap=idx + 64 + rows * w)  # intensities: half the pixels
    assert lb > 0 and ib == 0
