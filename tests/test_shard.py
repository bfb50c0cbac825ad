"""Band sharding (C5) of one image across ranks.

* CPU: the exchange plan of paper_2603_12016_b200/shard.py (table merge, halo
  plan, send/recv of halo rows) runs on 2 and 3 gloo ranks, with the C oracle
  computing each rank's owned ROIs; the concatenation equals the oracle's
  whole-image table bit for bit.
* GPU: the device path (fx_scan_accumulate / fx_label_table_copy /
  fx_featurize_owned) with 1..4 virtual bands in one process equals the
  single-call fx_featurize bit for bit.
"""
import os
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
GROUPS = ["intensity", "shape", "moments", "glcm", "glrlm", "glszm", "ngtdm"]


def straddling_image(h=150, w=120, seed=3):
    """Blobs placed on the band seams (rows 50, 75, 100) plus tall ROIs."""
    sys.path.insert(0, HERE)
    import inputs
    L = inputs.random_blobs((h, w), 30, seed=seed, max_r=14)
    L[10:140, 5:9] = 777          # spans every seam
    L[48:53, 60:70] = 778         # straddles row 50
    L[20, 100] = 779              # single pixel
    L[45:55, 110:118] = 778       # same label, second component across the seam
    I = inputs.uniform((h, w), seed)
    return I, L


class OracleBackend:
    """CPU stand-in for the device steps (scan, table, owned featurize)."""

    def __init__(self, params):
        from oracle import Oracle
        self.o, self.params = Oracle(), params
        self.cnt = self.bbox = None

    def tensor(self, values):
        return torch.tensor(values, dtype=torch.int64)

    def empty_rows(self, rows, width):
        return torch.zeros((rows, width), dtype=torch.int16)

    def empty_flat(self, n):
        return torch.zeros(n, dtype=torch.int16)

    def scan(self, I, L, oy):
        lab = L.numpy().view(np.uint16)
        cnt = np.zeros(65536, np.int64)
        bbox = np.zeros((4, 65536), np.int64)
        bbox[:2] = 0xFFFFFFFF
        labels, counts, bb = self.o.roi_table(lab)
        cnt[labels] = counts.astype(np.int64)
        bbox[0, labels] = bb[:, 0]
        bbox[1, labels] = bb[:, 1] + oy
        bbox[2, labels] = bb[:, 2]
        bbox[3, labels] = bb[:, 3] + oy
        return torch.from_numpy(cnt), torch.from_numpy(bbox)

    def set_table(self, cnt, bbox):
        self.cnt, self.bbox = cnt.numpy(), bbox.numpy()

    def featurize_owned(self, I, L, oy, y0, y1):
        lab, img = L.numpy().view(np.uint16), I.numpy().view(np.uint16)
        own = np.nonzero((self.cnt > 0) & (self.bbox[1] >= y0) & (self.bbox[1] < y1))[0]
        rows = []
        for l in own:
            ys, xs = np.nonzero(lab == l)
            assert len(ys) == self.cnt[l], "halo must hold the whole owned ROI"
            rows.append(self.o.roi_features(xs, ys + oy, img[ys, xs], GROUPS, self.params))
        return torch.tensor(own, dtype=torch.int64), torch.tensor(np.array(rows).reshape(len(own), -1))


def test_halo_rects_only_straddling_columns():
    """A tall ROI owned by band 0 moves only its own columns of bands 1-2; an ROI
    inside its band moves nothing (no full-width halo rows)."""
    from paper_2603_12016_b200 import shard
    bands = shard.band_plan(100, 4)
    cnt = np.zeros(65536, np.int64)
    bbox = np.zeros((4, 65536), np.int64)
    bbox[:2] = 0xFFFFFFFF
    for lab, (x0, y0, x1, y1) in {7: (10, 3, 19, 70), 9: (40, 30, 60, 45), 11: (0, 60, 99, 80)}.items():
        cnt[lab] = 5
        bbox[:, lab] = (x0, y0, x1, y1)
    rects = shard.halo_rects(cnt, bbox, bands)
    assert rects == [(0, 1, 25, 50, 10, 20), (0, 2, 50, 71, 10, 20), (2, 3, 75, 81, 0, 100)]


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, HERE)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import make_params
    from paper_2603_12016_b200 import shard
    I, L = straddling_image()
    H, W = L.shape
    y0, y1 = shard.band_plan(H, world)[rank]
    be = OracleBackend(make_params("default"))
    bI = torch.from_numpy(I[y0:y1].view(np.int16).copy())
    bL = torch.from_numpy(L[y0:y1].view(np.int16).copy())
    labels, values = shard.featurize_band(be, dist, rank, world, bI, bL, y0, H, W)
    q.put((rank, labels.numpy(), values.numpy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_band_sharding_matches_whole_image(oracle, world):
    from oracle import make_params
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + world * 7 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    labels = np.concatenate([r[1] for r in res])
    values = np.concatenate([r[2] for r in res])
    I, L = straddling_image()
    ol, ov = oracle.featurize(I, L, GROUPS, make_params("default"))
    order = np.argsort(labels)
    assert np.array_equal(labels[order], ol)
    assert np.array_equal(values[order], ov)


def _merge_worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2603_12016_b200 import shard
    out = []
    for n_labels in (50, 30000):  # sparse records, then the dense all-reduce
        rng = np.random.default_rng(1000 * rank + n_labels)
        cnt = np.zeros(65536, np.int64)
        bbox = np.zeros((4, 65536), np.int64)
        bbox[:2] = 0xFFFFFFFF
        labs = rng.choice(np.arange(1, 65536), n_labels, replace=False)
        cnt[labs] = rng.integers(1, 1000, n_labels)
        lo = rng.integers(0, 5000, (2, n_labels))
        bbox[:2, labs] = lo
        bbox[2:, labs] = lo + rng.integers(0, 100, (2, n_labels))
        c, b = shard.merge_tables(dist, torch.from_numpy(cnt.copy()), torch.from_numpy(bbox.copy()))
        rc, rb = torch.from_numpy(cnt.copy()), torch.from_numpy(bbox.copy())
        dist.all_reduce(rc, op=dist.ReduceOp.SUM)
        mins, maxs = rb[:2].contiguous(), rb[2:].contiguous()
        dist.all_reduce(mins, op=dist.ReduceOp.MIN)
        dist.all_reduce(maxs, op=dist.ReduceOp.MAX)
        out.append(bool(torch.equal(c, rc)) and bool(torch.equal(b, torch.cat([mins, maxs]))))
    q.put((rank, out))
    dist.barrier()
    dist.destroy_process_group()


def test_merge_tables_sparse_and_dense_agree():
    """The label-table merge: present-label records (few labels) and the dense
    all-reduce (many) give the identical merged table on every rank."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29700 + os.getpid() % 1000
    procs = [ctx.Process(target=_merge_worker, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(3)]
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    assert all(all(r[1]) for r in res), res


def test_halo_plan():
    from paper_2603_12016_b200 import shard
    bands = shard.band_plan(100, 4)
    assert bands == [(0, 25), (25, 50), (50, 75), (75, 100)]
    plan = shard.halo_transfers(bands, [30, 0, 5, 0])
    assert (1, 0, 25, 50) in plan and (2, 0, 50, 55) in plan and (3, 2, 75, 80) in plan
    cnt = np.zeros(65536, np.int64)
    bbox = np.zeros((4, 65536), np.int64)
    cnt[5], bbox[:, 5] = 10, (0, 20, 3, 61)
    assert shard.owned_need(cnt, bbox, 0, 25) == 37 and shard.owned_need(cnt, bbox, 25, 50) == 0


@pytest.mark.gpu
@pytest.mark.parametrize("nbands", [1, 2, 3, 4])
def test_device_band_sharding_bitwise(ctx, nbands):
    import ctypes as C
    import paper_2603_12016_b200 as fx
    from tools import synth
    from paper_2603_12016_b200 import fxg, shard
    I, L = straddling_image(200, 160, seed=9)
    big, _ = synth.packed_blob_mask_grid(256, 900, 40, 2)
    L = np.zeros((456, 256), np.uint16)
    L[:256] = big
    L[256:456, :160] = np.where(straddling_image(200, 160, seed=9)[1] > 0,
                                straddling_image(200, 160, seed=9)[1] + 100, 0)
    I = synth.uniform_u16(L.shape, 4)
    p = fx.resolve_profile("default")
    gl, gv = ctx.featurize(I, L, GROUPS, p)
    H, W = L.shape
    bands = shard.band_plan(H, nbands)
    lib = fxg.lib()
    mask = fx.resolve_groups(GROUPS)
    ncols = len(fx.feature_columns(mask, p))
    # 1: per-band scans (separate contexts = separate ranks)
    ctxs = [fx.Context(0) for _ in bands]
    tables = []
    for c, (y0, y1) in zip(ctxs, bands):
        bI, bL = np.ascontiguousarray(I[y0:y1]), np.ascontiguousarray(L[y0:y1])
        im = fxg.FxImage(bI.ctypes.data, bL.ctypes.data, W, y1 - y0, W, 0, y0, fxg.MEM_HOST)
        fxg._check(lib.fx_scan_accumulate(c.h, C.byref(im), 1))
        cnt = np.zeros(65536, np.uint64)
        bb = np.zeros((4, 65536), np.uint32)
        fxg._check(lib.fx_label_table_copy(c.h, cnt.ctypes.data_as(C.POINTER(C.c_uint64)),
                                           bb.ctypes.data_as(C.POINTER(C.c_uint32)), 0, 0))
        tables.append((cnt, bb))
    # 2: merge (what the NCCL all-reduce does)
    cnt = np.sum([t[0] for t in tables], axis=0).astype(np.uint64)
    bb = np.stack([t[1] for t in tables])
    merged = np.concatenate([bb[:, :2].min(0), bb[:, 2:].max(0)]).astype(np.uint32)
    rows_l, rows_v = [], []
    for c, (y0, y1) in zip(ctxs, bands):
        fxg._check(lib.fx_label_table_copy(c.h, cnt.ctypes.data_as(C.POINTER(C.c_uint64)),
                                           merged.ctypes.data_as(C.POINTER(C.c_uint32)), 1, 0))
        need = shard.owned_need(cnt.astype(np.int64), merged.astype(np.int64), y0, y1)
        eI = np.ascontiguousarray(I[y0:y1 + need])
        eL = np.ascontiguousarray(L[y0:y1 + need])
        im = fxg.FxImage(eI.ctypes.data, eL.ctypes.data, W, eL.shape[0], W, 0, y0, fxg.MEM_HOST)
        ol = np.zeros(65536, np.uint32)
        ov = np.zeros((65536, ncols))
        n = C.c_size_t()
        fxg._check(lib.fx_featurize_owned(c.h, C.byref(im), y0, y1, C.c_uint(mask), C.byref(p),
                                          ol.ctypes.data_as(C.POINTER(C.c_uint32)),
                                          ov.ctypes.data_as(C.POINTER(C.c_double)),
                                          C.c_size_t(65536), C.byref(n)))
        rows_l.append(ol[:n.value])
        rows_v.append(ov[:n.value])
    labels = np.concatenate(rows_l)
    values = np.concatenate(rows_v)
    order = np.argsort(labels)
    assert np.array_equal(labels[order], gl)
    assert np.array_equal(values[order], gv)
    for c in ctxs:
        c.close()


# ---- the library's own slide path over several devices (fx_multi_featurize_slide:
# table merge and straddling windows by peer reads) -------------------------

def _slide_image():
    """600 x 300: blob grid + seam straddlers + a ROI spanning every band (its
    halo exceeds the reserve rows: the separate band + halo raster path) + a
    two-component ROI split across the slide."""
    from tools import synth
    sys.path.insert(0, HERE)
    import inputs
    L = np.zeros((600, 300), np.uint16)
    g, _ = synth.packed_blob_mask_grid(300, 600, 64, 3)
    L[:300] = g
    L[300:600] = np.where(inputs.random_blobs((300, 300), 40, seed=5, max_r=30) > 0,
                          inputs.random_blobs((300, 300), 40, seed=5, max_r=30) + 200, 0)
    L[5:595, 140:143] = 900           # spans every band
    L[60:70, 10:20] = 901             # two components far apart
    L[520:530, 280:290] = 901
    L[140:170, 200:260] = 902         # straddles row 150
    I = synth.uniform_u16(L.shape, 8)
    return I, L


@pytest.mark.gpu
@pytest.mark.parametrize("devices", [[0], [0, 0], [0, 0, 0], [0, 0, 0, 0]])
def test_multi_slide_matches_single(ctx, devices):
    import paper_2603_12016_b200 as fx
    I, L = _slide_image()
    p = fx.resolve_profile("default")
    gl, gv = ctx.featurize(I, L, GROUPS, p)
    m = fx.Multi(devices)
    try:
        ml, mv = m.featurize_slide(I, L, GROUPS, p, origin=(0, 0))
        # twice: the contexts' tables and buffers are left reusable
        ml2, mv2 = m.featurize_slide(I, L, GROUPS, p)
    finally:
        m.close()
    assert np.array_equal(gl, ml) and np.array_equal(gv, mv)
    assert np.array_equal(ml, ml2) and np.array_equal(mv, mv2)


@pytest.mark.gpu
def test_multi_slide_c5_shape(ctx):
    """C5-like 16384^2 slide of ~2e5-px ROIs over 4 contexts == one featurize."""
    import paper_2603_12016_b200 as fx
    from tools import synth
    L, _ = synth.packed_blob_mask_grid(16384, 200000, 576, 1)
    L = np.roll(L, 340, axis=0)
    I = synth.uniform_u16(L.shape, 5)
    groups = ["intensity", "moments", "glcm"]
    p = fx.resolve_profile("default")
    gl, gv = ctx.featurize(I, L, groups, p)
    m = fx.Multi([0, 0, 0, 0])
    try:
        ml, mv = m.featurize_slide(I, L, groups, p)
    finally:
        m.close()
    assert np.array_equal(gl, ml) and np.array_equal(gv, mv)


# ---- the device backend itself with 2 ranks: two processes on one GPU, the
# collectives staged through host memory over gloo (the ranks' kernels never
# wait on each other) ----------------------------------------------------------

class StagedDist:
    """torch.distributed over gloo for CUDA tensors: every collective / p2p op
    copies through host memory.  Exposes the subset shard.featurize_band uses."""
    ReduceOp = dist.ReduceOp

    class P2POp:
        def __init__(self, op, tensor, peer):
            self.op, self.tensor, self.peer = op, tensor, peer

    isend, irecv = "isend", "irecv"

    @staticmethod
    def get_world_size():
        return dist.get_world_size()

    @staticmethod
    def all_reduce(t, op=dist.ReduceOp.SUM):
        c = t.cpu()
        dist.all_reduce(c, op=op)
        t.copy_(c)

    @staticmethod
    def all_gather(outs, t):
        cs = [torch.empty_like(o, device="cpu") for o in outs]
        dist.all_gather(cs, t.cpu())
        for o, c in zip(outs, cs):
            o.copy_(c)

    @staticmethod
    def batch_isend_irecv(ops):
        reqs, backs = [], []
        for o in ops:
            if o.op == "isend":
                reqs.append(dist.isend(o.tensor.cpu(), o.peer))
            else:
                buf = torch.empty_like(o.tensor, device="cpu")
                reqs.append(dist.irecv(buf, o.peer))
                backs.append((o.tensor, buf))

        class Done:
            def wait(self_):
                for r in reqs:
                    r.wait()
                for t, b in backs:
                    t.copy_(b)
        return [Done()]


def _device_worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, HERE)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2603_12016_b200 as fx
    from paper_2603_12016_b200 import shard
    I, L = _slide_image()
    H, W = L.shape
    y0, y1 = shard.band_plan(H, world)[rank]
    ctx = fx.Context(0)
    be = shard.DeviceBackend(ctx, GROUPS, fx.resolve_profile("default"))
    bI = torch.from_numpy(I[y0:y1].view(np.int16).copy()).cuda()
    bL = torch.from_numpy(L[y0:y1].view(np.int16).copy()).cuda()
    labels, values = shard.featurize_band(be, StagedDist, rank, world, bI, bL, y0, H, W)
    q.put((rank, labels.cpu().numpy(), values.cpu().numpy()))
    dist.barrier()
    ctx.close()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_device_backend_multi_rank(ctx, world):
    import paper_2603_12016_b200 as fx
    mpc = mp.get_context("spawn")
    q = mpc.Queue()
    port = 29700 + world * 11 + os.getpid() % 1000
    procs = [mpc.Process(target=_device_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    labels = np.concatenate([r[1] for r in res]).astype(np.uint32)
    values = np.concatenate([r[2] for r in res])
    order = np.argsort(labels)
    I, L = _slide_image()
    gl, gv = ctx.featurize(I, L, GROUPS, fx.resolve_profile("default"))
    assert np.array_equal(labels[order], gl)
    assert np.array_equal(values[order], gv)


def test_halo_rows_travel_as_bytes():
    """NCCL has no int16: the halo rows are exchanged as uint8 views."""
    import inspect
    from paper_2603_12016_b200 import shard
    src = inspect.getsource(shard.featurize_band)
    assert "view(torch.uint8)" in src
