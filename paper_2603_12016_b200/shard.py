"""Row-band sharding of one large image across ranks (C5).

One process per GPU.  Rank k owns image rows [y0_k, y1_k).  The exchange steps,
all through torch.distributed (NCCL on GPUs, gloo in the CPU tests):

1. local label scan of the own band into a label table in global coordinates;
2. merge of the partial tables (the mergeable accumulators): count = SUM,
   xmin/ymin = MIN, xmax/ymax = MAX -- the present labels' records all-gathered
   when the bands hold few labels, else a dense all-reduce per array; integer-
   exact, so the merged table is bit-identical to a whole-image scan;
3. ownership: a ROI belongs to the band that holds its first row (ymin);
4. halo: an owner needs, for each owned ROI that runs below its band, that ROI's
   window columns in the rows below the band (halo_rects, the same plan on every
   rank from the merged table); the ranks holding those rows send the rectangles,
   one packed message per (source, owner) and raster -- only straddling windows
   move, never whole rows, so a tall or slide-spanning ROI costs its own columns;
5. each rank featurizes its owned ROIs on band + halo.  Non-mergeable statistics
   (order statistics, the contour edge set) need no merge: the owner holds the
   whole window.  Rows are therefore identical to a single-GPU featurize of the
   whole image, for any number of bands.

The device backend drives libfxg (fx_scan_accumulate, fx_label_table_copy,
fx_featurize_owned); tests/test_shard.py drives the same plan with the C oracle
on CPU ranks over gloo.
"""
from __future__ import annotations

import numpy as np

NL = 65536
SENT = 0xFFFFFFFF


def band_plan(height: int, world: int):
    """Equal row bands [y0, y1) per rank (the last absorbs the remainder)."""
    base = height // world
    return [(k * base, height if k == world - 1 else (k + 1) * base) for k in range(world)]


def owned_need(cnt, bbox, y0, y1):
    """Rows past y1 needed by the ROIs owned by band [y0, y1): max(ymax)+1 - y1, >= 0."""
    ymin, ymax = bbox[1], bbox[3]
    own = (cnt > 0) & (ymin >= y0) & (ymin < y1)
    if not own.any():
        return 0
    return max(0, int(ymax[own].max()) + 1 - y1)


def halo_transfers(bands, needs):
    """(src, dst, row_lo, row_hi) for every halo slice: rank dst needs rows
    [y1_dst, y1_dst + need_dst), held by the ranks whose bands intersect them."""
    out = []
    for dst, ((_, y1), need) in enumerate(zip(bands, needs)):
        lo, hi = y1, y1 + int(need)
        for src, (b0, b1) in enumerate(bands):
            a, b = max(lo, b0), min(hi, b1)
            if a < b:
                out.append((src, dst, a, b))
    return out


def len_world(dist):
    return dist.get_world_size()


def halo_rects(cnt, bbox, bands):
    """(dst, src, row_lo, row_hi, x_lo, x_hi) for every owned ROI that runs below its
    owner's band: its window columns in the rows below, split by the bands holding
    them.  Ordered by owner, label, source: every rank derives the same list."""
    cnt, bbox = np.asarray(cnt), np.asarray(bbox)
    xmin, ymin, xmax, ymax = (bbox[i].astype(np.int64) for i in range(4))
    present = cnt > 0
    out = []
    for dst, (b0, b1) in enumerate(bands):
        own = np.nonzero(present & (ymin >= b0) & (ymin < b1) & (ymax >= b1))[0]
        for lab in own:
            lo, hi = b1, int(ymax[lab]) + 1
            for src, (s0, s1) in enumerate(bands):
                a, b = max(lo, s0), min(hi, s1)
                if a < b:
                    out.append((dst, src, a, b, int(xmin[lab]), int(xmax[lab]) + 1))
    return out


def merge_tables(dist, cnt, bbox):
    """Merge of the partial label tables (torch tensors, int64): cnt [65536] SUM;
    bbox [4, 65536] = xmin, ymin (MIN), xmax, ymax (MAX).  A band holding few
    labels sends only its present labels' records (label, count, box: 48 B each,
    all-gathered); a band holding many all-reduces the dense arrays (2.5 MB).
    Integer-exact either way: the merged table is identical."""
    import torch
    k = int((cnt > 0).sum().item())
    ks = [torch.zeros(1, dtype=torch.int64, device=cnt.device) for _ in range(len_world(dist))]
    dist.all_gather(ks, torch.tensor([k], dtype=torch.int64, device=cnt.device))
    kmax = max(int(t.item()) for t in ks)
    if kmax * 6 * 8 * len(ks) < 3 * NL * 8:  # sparse records beat the dense all-reduce
        labs = torch.nonzero(cnt > 0).squeeze(1)
        rec = torch.full((kmax, 6), -1, dtype=torch.int64, device=cnt.device)
        rec[:k, 0] = labs
        rec[:k, 1] = cnt[labs]
        rec[:k, 2:] = bbox[:, labs].t()
        recs = [torch.empty_like(rec) for _ in ks]
        dist.all_gather(recs, rec)
        allr = torch.cat(recs)
        allr = allr[allr[:, 0] >= 0]
        lab = allr[:, 0]
        cnt = torch.zeros(NL, dtype=torch.int64, device=cnt.device).index_add_(0, lab, allr[:, 1])
        mins = torch.full((2, NL), SENT, dtype=torch.int64, device=cnt.device)
        maxs = torch.zeros((2, NL), dtype=torch.int64, device=cnt.device)
        for r in range(2):
            mins[r].scatter_reduce_(0, lab, allr[:, 2 + r], reduce="amin", include_self=True)
            maxs[r].scatter_reduce_(0, lab, allr[:, 4 + r], reduce="amax", include_self=True)
        return cnt, torch.cat([mins, maxs])
    dist.all_reduce(cnt, op=dist.ReduceOp.SUM)
    mins, maxs = bbox[:2].contiguous(), bbox[2:].contiguous()
    dist.all_reduce(mins, op=dist.ReduceOp.MIN)
    dist.all_reduce(maxs, op=dist.ReduceOp.MAX)
    bbox[:2] = mins
    bbox[2:] = maxs
    return cnt, bbox


def featurize_band(backend, dist, rank, world, band_intensity, band_labels, y0, height,
                   width):
    """Runs steps 1-5 for this rank.  band_* are [y1-y0, width] arrays/tensors of
    the rank's own rows.  Returns (labels, values) of the ROIs this rank owns."""
    import torch

    bands = band_plan(height, world)
    assert bands[rank][0] == y0
    y1 = bands[rank][1]
    # 1-2: scan + merge
    cnt, bbox = backend.scan(band_intensity, band_labels, y0)
    cnt, bbox = merge_tables(dist, cnt, bbox)
    backend.set_table(cnt, bbox)
    # 3-4: halo plan from the merged table (on the host: 1.5 MB), identical on every rank
    hc, hb = cnt.cpu().numpy(), bbox.cpu().numpy()
    rects = halo_rects(hc, hb, bands)
    need = max([r[3] - y1 for r in rects if r[0] == rank], default=0)
    ext_rows = (y1 - y0) + need
    ext_I = backend.empty_rows(ext_rows, width)
    ext_L = backend.empty_rows(ext_rows, width)
    ext_I[: y1 - y0] = band_intensity
    ext_L[: y1 - y0] = band_labels
    ext_I[y1 - y0:] = 0  # outside the rectangles: no pixel of any owned ROI
    ext_L[y1 - y0:] = 0
    ops, recvs = [], []
    # rows travel as bytes: NCCL has no 16-bit integer type (torch's NCCL type map
    # lacks int16), so the uint16 rasters are viewed as uint8 on both sides
    as_bytes = lambda t: t.contiguous().view(torch.uint8)
    for other in range(world):
        if other == rank:
            continue
        out_r = [r for r in rects if r[1] == rank and r[0] == other]
        if out_r:  # my rows of the owner's straddling windows, one message per raster
            for band in (band_intensity, band_labels):
                parts = [band[a - y0:b - y0, xl:xh].reshape(-1) for _, _, a, b, xl, xh in out_r]
                ops.append(dist.P2POp(dist.isend, as_bytes(torch.cat(parts)), other))
        in_r = [r for r in rects if r[0] == rank and r[1] == other]
        if in_r:
            total = sum((b - a) * (xh - xl) for _, _, a, b, xl, xh in in_r)
            bufs = [backend.empty_flat(total), backend.empty_flat(total)]
            for buf in bufs:
                ops.append(dist.P2POp(dist.irecv, buf.view(torch.uint8), other))
            recvs.append((in_r, bufs))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    for in_r, (bI, bL) in recvs:  # the rectangles into the extended rasters
        at = 0
        for _, _, a, b, xl, xh in in_r:
            k = (b - a) * (xh - xl)
            ext_I[a - y0:b - y0, xl:xh] = bI[at:at + k].view(b - a, xh - xl)
            ext_L[a - y0:b - y0, xl:xh] = bL[at:at + k].view(b - a, xh - xl)
            at += k
    # 5: featurize owned ROIs on band + halo
    return backend.featurize_owned(ext_I, ext_L, y0, y0, y1)


class DeviceBackend:
    """libfxg on this rank's GPU; tensors are torch CUDA tensors (NCCL)."""

    def __init__(self, ctx, groups, params):
        import torch

        from . import fxg
        self.torch, self.fxg, self.ctx = torch, fxg, ctx
        self.groups, self.params = groups, params
        self.mask = groups if isinstance(groups, int) else fxg.resolve_groups(list(groups))
        self.ncols = len(fxg.feature_columns(self.mask, params))

    def tensor(self, values):
        return self.torch.tensor(values, dtype=self.torch.int64, device="cuda")

    def empty_rows(self, rows, width):
        return self.torch.empty((rows, width), dtype=self.torch.int16, device="cuda")

    def empty_flat(self, n):
        return self.torch.empty(n, dtype=self.torch.int16, device="cuda")

    def _image(self, I, L, oy):
        h, w = L.shape
        return self.fxg.FxImage(I.data_ptr(), L.data_ptr(), w, h, w, 0, oy, self.fxg.MEM_DEVICE)

    def scan(self, I, L, oy):
        import ctypes as C
        lib = self.fxg.lib()
        im = self._image(I, L, oy)
        self.fxg._check(lib.fx_scan_accumulate(self.ctx.h, C.byref(im), 1))
        cnt = self.torch.empty(NL, dtype=self.torch.int64, device="cuda")
        bb = self.torch.empty((4, NL), dtype=self.torch.int32, device="cuda")
        self.fxg._check(lib.fx_label_table_copy(self.ctx.h, C.c_void_p(cnt.data_ptr()),
                                                C.c_void_p(bb.data_ptr()), 0, self.fxg.MEM_DEVICE))
        return cnt, bb.to(self.torch.int64) & SENT

    def set_table(self, cnt, bbox):
        import ctypes as C
        bb = bbox.to(self.torch.int32).contiguous()
        cnt = cnt.contiguous()
        self.fxg._check(self.fxg.lib().fx_label_table_copy(
            self.ctx.h, C.c_void_p(cnt.data_ptr()), C.c_void_p(bb.data_ptr()), 1,
            self.fxg.MEM_DEVICE))

    def featurize_owned(self, I, L, oy, own_y0, own_y1):
        import ctypes as C
        cap = NL
        out_l = self.torch.empty(cap, dtype=self.torch.int32, device="cuda")
        out_v = self.torch.empty((cap, self.ncols), dtype=self.torch.float64, device="cuda")
        im = self._image(I, L, oy)
        n = C.c_size_t()
        self.fxg._check(self.fxg.lib().fx_featurize_owned(
            self.ctx.h, C.byref(im), own_y0, own_y1, C.c_uint(self.mask), C.byref(self.params),
            C.c_void_p(out_l.data_ptr()), C.c_void_p(out_v.data_ptr()), C.c_size_t(cap),
            C.byref(n)))
        k = n.value
        return out_l[:k], out_v[:k]
