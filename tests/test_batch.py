"""Batch path (C4: many image pairs per call, fx_featurize_batch).

Every image of a batch must give exactly the rows fx_featurize gives for it alone
(bit-exact), whatever the batch composition: mixed sizes, heights that are not a
multiple of the 64-row scan strip, origins, empty images, more images than one
launch set holds (128 slots), host or device rasters, stacked device tensors read
in place.  The single-image rows are themselves pinned to the oracle by
test_gpu_parity.py; one case here also checks a batch against the oracle directly.
"""
import ctypes as C
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import inputs  # noqa: E402
from parity import assert_parity  # noqa: E402

GROUPS = ["intensity", "shape", "moments", "glcm", "glrlm", "glszm", "ngtdm"]


def _pairs(specs, seed=0):
    out = []
    for k, (h, w, n) in enumerate(specs):
        L = inputs.random_blobs((h, w), n, seed=seed + k, max_r=min(h, w) // 4 + 1) if n else \
            np.zeros((h, w), np.uint16)
        I = inputs.uniform((h, w), seed + 100 + k)
        out.append((I, L))
    return out


def _check_same(ctx, pairs, res, params, origins=None):
    assert len(res) == len(pairs)
    for k, ((I, L), (bl, bv)) in enumerate(zip(pairs, res)):
        o = origins[k] if origins is not None else (0, 0)
        sl, sv = ctx.featurize(I, L, GROUPS, params, origin=o)
        assert np.array_equal(bl, sl), k
        assert np.array_equal(bv, sv), k


@pytest.mark.gpu
def test_batch_mixed_sizes_bitwise(ctx):
    import paper_2603_12016_b200 as fx
    p = fx.resolve_profile("default")
    specs = [(100, 90, 12), (64, 64, 5), (1, 1, 0), (37, 200, 9), (130, 61, 15), (10, 10, 0),
             (256, 256, 40), (65, 300, 20)]
    pairs = _pairs(specs, seed=11)
    pairs[2] = (np.array([[7]], np.uint16), np.array([[3]], np.uint16))  # one-pixel image
    # labels spread over many 1024-label compaction blocks, up to 65535
    pairs[4] = (pairs[4][0], inputs.random_blobs((130, 61), 15, seed=4, max_r=12,
                                                 label_values=[1500, 40000, 65535, 2049, 1024]))
    origins = [(k * 13, 1000 + k * 7) for k in range(len(pairs))]
    res = ctx.featurize_batch(pairs, GROUPS, p, origins=origins)
    _check_same(ctx, pairs, res, p, origins)


@pytest.mark.gpu
def test_batch_vs_oracle(ctx, oracle):
    import paper_2603_12016_b200 as fx
    from oracle import make_params
    p = make_params("default")
    cols = fx.feature_columns(GROUPS, fx.resolve_profile("default"))
    pairs = _pairs([(120, 140, 10), (77, 50, 6), (200, 64, 14)], seed=5)
    res = ctx.featurize_batch(pairs, GROUPS, fx.resolve_profile("default"))
    for (I, L), (bl, bv) in zip(pairs, res):
        ol, ov = oracle.featurize(I, L, GROUPS, p)
        assert_parity(cols, bl, bv, ol, ov, I, L)


@pytest.mark.gpu
def test_batch_more_than_one_launch_set(ctx):
    """1,100 images > 512 slots: three sub-batches, staged double-buffered."""
    import paper_2603_12016_b200 as fx
    p = fx.resolve_profile("performance")
    specs = [(48 + (k % 5) * 16, 40 + (k % 7) * 8, 1 + k % 6) for k in range(1100)]
    pairs = _pairs(specs, seed=21)
    res = ctx.featurize_batch(pairs, GROUPS, p)
    _check_same(ctx, pairs, res, p)
    # the context stays usable for single calls afterwards (table left clean)
    I, L = pairs[7]
    sl, sv = ctx.featurize(I, L, GROUPS, p)
    assert np.array_equal(res[7][0], sl) and np.array_equal(res[7][1], sv)


@pytest.mark.gpu
def test_batch_all_empty_and_empty_list(ctx):
    import paper_2603_12016_b200 as fx
    p = fx.resolve_profile("default")
    assert ctx.featurize_batch([], GROUPS, p) == []
    pairs = _pairs([(50, 50, 0), (20, 70, 0)])
    res = ctx.featurize_batch(pairs, GROUPS, p)
    assert [len(r[0]) for r in res] == [0, 0]


@pytest.mark.gpu
def test_batch_capacity_error(ctx):
    import paper_2603_12016_b200 as fx
    p = fx.resolve_profile("default")
    pairs = _pairs([(100, 100, 10), (100, 100, 10)], seed=3)
    with pytest.raises(fx.FxError) as e:
        ctx.featurize_batch(pairs, GROUPS, p, cap_rois=5)
    assert e.value.code == 10
    res = ctx.featurize_batch(pairs, GROUPS, p)  # recovers
    _check_same(ctx, pairs, res, p)


def _device_batch(ctx, tI, tL, views, p, mask, ncols, cap):
    import torch
    from paper_2603_12016_b200 import fxg
    ims = (fxg.FxImage * len(views))()
    for k, (vi, vl) in enumerate(views):
        h, w = vl.shape
        ims[k] = fxg.FxImage(vi.data_ptr(), vl.data_ptr(), w, h, vl.stride(0), 0, 0,
                             fxg.MEM_DEVICE)
    out_l = torch.zeros(cap, dtype=torch.int32, device="cuda")
    out_v = torch.zeros((cap, ncols), dtype=torch.float64, device="cuda")
    offs = ctx.featurize_batch_raw(ims, len(views), mask, p, out_l.data_ptr(), out_v.data_ptr(),
                                   cap)
    torch.cuda.synchronize()
    return out_l.cpu().numpy().view(np.uint32), out_v.cpu().numpy(), offs


@pytest.mark.gpu
@pytest.mark.parametrize("stacked", [True, False])
def test_batch_device_rasters(ctx, stacked):
    """[T, 192, 160] device stack read in place (stacked) or separate tensors (staged)."""
    import torch
    import paper_2603_12016_b200 as fx
    p = fx.resolve_profile("default")
    mask = fx.resolve_groups(GROUPS)
    ncols = len(fx.feature_columns(mask, p))
    T, H, W = 9, 192, 160
    pairs = _pairs([(H, W, 8 + k) for k in range(T)], seed=31)
    if stacked:
        tI = torch.from_numpy(np.stack([a for a, _ in pairs]).view(np.int16)).cuda()
        tL = torch.from_numpy(np.stack([b for _, b in pairs]).view(np.int16)).cuda()
        views = [(tI[k], tL[k]) for k in range(T)]
    else:
        views = [(torch.from_numpy(a.view(np.int16)).cuda(), torch.from_numpy(b.view(np.int16)).cuda())
                 for a, b in pairs]
        tI = tL = None
    cap = 4096
    bl, bv, offs = _device_batch(ctx, tI, tL, views, p, mask, ncols, cap)
    for k, (I, L) in enumerate(pairs):
        sl, sv = ctx.featurize(I, L, GROUPS, p)
        assert np.array_equal(bl[offs[k]:offs[k + 1]], sl), k
        assert np.array_equal(bv[offs[k]:offs[k + 1]], sv), k


@pytest.mark.gpu
def test_batch_host_stack_packed(ctx):
    """A host [T, H, W] stack is one run of back-to-back images: it is
    packed in 4096-row blocks (a block boundary falls inside an image), noise tiles
    fall back to raw rows, and every image's rows equal its device-resident call."""
    import paper_2603_12016_b200 as fx
    from paper_2603_12016_b200 import fxg
    p = fx.resolve_profile("default")
    mask = fx.resolve_groups(GROUPS)
    T, H, W = 44, 128, 192
    pairs = _pairs([(H, W, 6 + k % 9) for k in range(T)], seed=17)
    rng = np.random.default_rng(3)
    for k in (5, 6, 40):  # label noise: these rows do not pack
        pairs[k] = (pairs[k][0], rng.integers(0, 65536, (H, W)).astype(np.uint16))
    sI = np.ascontiguousarray(np.stack([a for a, _ in pairs]))
    sL = np.ascontiguousarray(np.stack([b for _, b in pairs]))
    ims = (fxg.FxImage * T)()
    for k in range(T):
        ims[k] = fxg.FxImage(sI[k].ctypes.data, sL[k].ctypes.data, W, H, W, 0, 0, fxg.MEM_HOST)
    cap = int(sum(np.count_nonzero(np.bincount(L.ravel(), minlength=65536)[1:]) for _, L in pairs))
    try:
        ctx.set_packing(True)
        bl, bv, offs = ctx.featurize_batch_raw(ims, T, mask, p, None, None, cap)
        pk, _ = ctx.last_transfer()
        ctx.set_packing(False)
        rl, rv, roffs = ctx.featurize_batch_raw(ims, T, mask, p, None, None, cap)
        raw, _ = ctx.last_transfer()
    finally:
        ctx.set_packing(True)
    assert raw == T * H * W * 4 and pk < 0.8 * raw, (pk, raw)
    assert np.array_equal(offs, roffs) and np.array_equal(bl, rl) and np.array_equal(bv, rv)
    for k in (0, 5, 31, 32, 40, 43):  # 32: straddles the 4096-row block boundary
        sl, sv = ctx.featurize(sI[k], sL[k], GROUPS, p)
        assert np.array_equal(bl[offs[k]:offs[k + 1]], sl), k
        assert np.array_equal(bv[offs[k]:offs[k + 1]], sv), k


# ---- banded host path (fx_featurize with host rasters: H2D / kernels / D2H
# overlapped in row bands) must give exactly the unbanded rows ---------------

@pytest.mark.gpu
@pytest.mark.parametrize("rows", [64, 128, 512])
def test_banded_host_path_bitwise(ctx, rows):
    import paper_2603_12016_b200 as fx
    p = fx.resolve_profile("default")
    # multi-component ROIs spanning many bands, holes, border contact, big windows
    L = inputs.random_blobs((700, 300), 90, seed=7, max_r=40,
                            label_values=np.array([1, 2, 3, 65535, 40000, 17, 900]))
    L[650:700, 0:300:7] = 5  # one ROI spread over a wide strip of the bottom band
    I = inputs.uniform(L.shape, 3)
    try:
        ctx.set_band_rows(-1)
        rl, rv = ctx.featurize(I, L, GROUPS, p)
        ctx.set_band_rows(rows)
        bl, bv = ctx.featurize(I, L, GROUPS, p)
    finally:
        ctx.set_band_rows(0)
    assert np.array_equal(rl, bl)
    assert np.array_equal(rv, bv)


def _packed_case(name):
    rng = np.random.default_rng(5)
    if name == "blobs":
        L = inputs.random_blobs((700, 300), 90, seed=7, max_r=40,
                                label_values=np.array([1, 2, 3, 65535, 40000, 17, 900]))
    elif name == "noise_rows":  # some blocks do not pack into half their size: sent raw
        L = inputs.random_blobs((900, 256), 60, seed=3, max_r=30)
        L[300:700] = rng.integers(0, 65536, (400, 256)).astype(np.uint16)
    elif name == "odd_width":  # width not a multiple of 8 / 32; labels on the last column
        L = inputs.random_blobs((520, 333), 50, seed=9, max_r=25)
        L[:, 332] = 7
        L[100:110, :] = 11
    elif name == "full_rows":  # labelled everywhere: every intensity crosses
        L = inputs.random_labels((400, 192), 20, seed=4, p_bg=0.0)
    elif name == "wide_odd":  # three 2048-px unpack tiles, the last partial; runs across tiles
        L = inputs.random_blobs((260, 4100), 120, seed=12, max_r=35)
        L[:, 2040:2060] = 3
        L[50:60, 4090:] = 4
    else:  # empty
        L = np.zeros((300, 130), np.uint16)
    return inputs.uniform(L.shape, 11), L


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["blobs", "noise_rows", "odd_width", "full_rows", "wide_odd", "empty"])
def test_packed_host_path_bitwise(ctx, oracle, name):
    """Banded host rasters crossing PCIe packed (label change points + labelled
    intensities, host threads) == raw bands == the unbanded call, bit for bit, and
    the oracle; raw fallback per block where the labels do not pack."""
    import paper_2603_12016_b200 as fx
    from oracle import make_params as oparams
    p = fx.resolve_profile("default")
    I, L = _packed_case(name)
    try:
        ctx.set_band_rows(-1)
        rl, rv = ctx.featurize(I, L, GROUPS, p)
        ctx.set_band_rows(128)
        ctx.set_packing(False)
        bl, bv = ctx.featurize(I, L, GROUPS, p)
        raw_h2d, _ = ctx.last_transfer()
        ctx.set_packing(True)
        pl, pv = ctx.featurize(I, L, GROUPS, p)
        pk_h2d, _ = ctx.last_transfer()
        pl2, pv2 = ctx.featurize(I, L, GROUPS, p)  # staging buffers reused
    finally:
        ctx.set_band_rows(0)
        ctx.set_packing(True)
    assert raw_h2d == 2 * L.size * 2
    if name in ("blobs", "odd_width", "wide_odd", "empty"):  # a share of the blocks always goes raw
        assert pk_h2d < 0.75 * raw_h2d, (pk_h2d, raw_h2d)
    for a, b in ((rl, bl), (rl, pl), (rl, pl2)):
        assert np.array_equal(a, b)
    for a, b in ((rv, bv), (rv, pv), (rv, pv2)):
        assert np.array_equal(a, b)
    ol, ov = oracle.featurize(I, L, GROUPS, oparams("default"))
    assert_parity(fx.feature_columns(GROUPS, p), pl, pv, ol, ov, I, L)


@pytest.mark.gpu
def test_packed_host_path_concurrent_contexts(ctx):
    """Two contexts packing at once from two host threads (one process-wide packer
    pool, taken in turn): each gets the unbanded rows."""
    import threading
    import paper_2603_12016_b200 as fx
    p = fx.resolve_profile("default")
    cases = [_packed_case("blobs"), _packed_case("odd_width")]
    ctx.set_band_rows(-1)
    try:
        want = [ctx.featurize(I, L, GROUPS, p) for I, L in cases]
    finally:
        ctx.set_band_rows(0)
    ctxs = [fx.Context(0), fx.Context(0)]
    got = [[None] * 4, [None] * 4]
    errs = []

    def run(t):
        try:
            ctxs[t].set_band_rows(128)
            for k in range(4):
                got[t][k] = ctxs[t].featurize(*cases[(t + k) % 2], GROUPS, p)
        except Exception as e:  # surfaced below
            errs.append(e)

    th = [threading.Thread(target=run, args=(t,)) for t in range(2)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    for c in ctxs:
        c.close()
    assert not errs, errs
    for t in range(2):
        for k in range(4):
            wl, wv = want[(t + k) % 2]
            gl, gv = got[t][k]
            assert np.array_equal(wl, gl) and np.array_equal(wv, gv), (t, k)


@pytest.mark.gpu
def test_banded_host_path_c2_bitwise(ctx):
    """bench.py's e2e call (host rasters, automatic bands) == the device-resident call"""
    import torch
    import bench
    import paper_2603_12016_b200 as fx
    I, L, _ = bench.workload(0)
    p = fx.resolve_profile(bench.PROFILE)
    mask = fx.resolve_groups(bench.GROUPS)
    ncols = len(fx.feature_columns(mask, p))
    h, w = L.shape
    n = bench.ROI_COUNT
    dI = torch.from_numpy(I.view(np.int16)).cuda()
    dL = torch.from_numpy(L.view(np.int16)).cuda()
    ol = torch.empty(n, dtype=torch.int32, device="cuda")
    ov = torch.empty((n, ncols), dtype=torch.float64, device="cuda")
    assert ctx.featurize_device(dI.data_ptr(), dL.data_ptr(), w, h, w, mask, p, ol.data_ptr(),
                                ov.data_ptr(), n) == n
    hI = torch.from_numpy(I.view(np.int16)).pin_memory()
    hL = torch.from_numpy(L.view(np.int16)).pin_memory()
    hv = torch.empty((n, ncols), dtype=torch.float64).pin_memory()
    hl = torch.empty(n, dtype=torch.int32).pin_memory()
    assert ctx.featurize_host_ptrs(hI.data_ptr(), hL.data_ptr(), w, h, mask, p, hl.data_ptr(),
                                   hv.data_ptr(), n) == n
    assert torch.equal(hl, ol.cpu())
    assert torch.equal(hv, ov.cpu())


# ---- several devices of one process (fx_multi): rows identical to one context --

@pytest.mark.gpu
@pytest.mark.parametrize("devices", [[0], [0, 0], [0, 0, 0]])
def test_multi_batch_matches_single(ctx, devices):
    """Chunks of 512 images dealt over the contexts (the same GPU listed several
    times stands in for several devices: each context has its own streams, buffers
    and host thread); output order and values identical to fx_featurize_batch."""
    import paper_2603_12016_b200 as fx
    p = fx.resolve_profile("default")
    specs = [(48 + (k % 5) * 16, 40 + (k % 7) * 8, (k % 6)) for k in range(1300)]
    pairs = _pairs(specs, seed=31)
    ref = ctx.featurize_batch(pairs, GROUPS, p)
    m = fx.Multi(devices)
    try:
        res = m.featurize_batch(pairs, GROUPS, p)
    finally:
        m.close()
    assert len(res) == len(ref)
    for (rl, rv), (ml, mv) in zip(ref, res):
        assert np.array_equal(rl, ml)
        assert np.array_equal(rv, mv)


@pytest.mark.gpu
def test_multi_batch_capacity_error(ctx):
    import paper_2603_12016_b200 as fx
    p = fx.resolve_profile("performance")
    pairs = _pairs([(64, 64, 6)] * 700, seed=3)
    m = fx.Multi([0, 0])
    try:
        with pytest.raises(fx.FxError) as e:
            m.featurize_batch(pairs, GROUPS, p, cap_rois=10)
        assert e.value.kind == "CapacityError"
        # the contexts stay usable
        res = m.featurize_batch(pairs[:50], GROUPS, p)
        assert len(res) == 50
    finally:
        m.close()
