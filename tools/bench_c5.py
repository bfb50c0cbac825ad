#!/usr/bin/env python3
"""C5 workload (BASELINE.json configs[4]): a 65536 x 65536 uint16 whole-slide
image with large blob ROIs.

Labels: blob_mask_grid(8192, 200000, 144, seed 1) (12 x 12 blobs of ~1.2e5 px),
replicated 8 x 8 with distinct label ranges (9216 ROIs), rolled down by 4096 rows
so blobs straddle every 8192-row band seam (the wrapped top/bottom blobs become
two-component ROIs).  Intensities: a counter hash of the pixel index, so any row
band can be generated on its own GPU and equals the same rows of the whole image.

  python tools/bench_c5.py                  # one fx_featurize on the whole slide
  torchrun --nproc-per-node N tools/bench_c5.py --sharded
      # row bands over N GPUs: local scan, NCCL table merge, halo exchange,
      # owned-ROI featurize (paper_2603_12016_b200/shard.py); time = max over ranks
Prints one JSON line (rank 0).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def band_rasters(torch, dev, tile_lab, per, S, T, y0, y1, chunk=1024, roll=None):
    """Rows [y0, y1) of the rolled composition: labels and hashed intensities
    (built in row chunks to bound the int64 temporaries)."""
    k = S // T
    I = torch.empty((y1 - y0, S), dtype=torch.int16, device=dev)
    L = torch.empty((y1 - y0, S), dtype=torch.int16, device=dev)
    cols = torch.arange(S, device=dev, dtype=torch.int64)
    bx, tx = cols // T, cols % T
    for c0 in range(y0, y1, chunk):
        c1 = min(y1, c0 + chunk)
        rows = torch.arange(c0, c1, device=dev, dtype=torch.int64)
        src = (rows - (T // 2 if roll is None else roll)) % S  # row of the unrolled composition
        by, ty = src // T, src % T                 # tile block row, row inside the tile
        lab = tile_lab[ty][:, tx]
        off = (by[:, None] * k + bx[None, :]) * per
        L[c0 - y0:c1 - y0] = torch.where(lab > 0, lab + off, torch.zeros_like(lab)).to(torch.int32).to(torch.int16)
        idx = rows[:, None] * S + cols[None, :]
        h = (idx * 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFF
        h = (h ^ (h >> 29)) * 0xBF58476D1CE4E5B9 & 0xFFFFFFFFFFFF
        I[c0 - y0:c1 - y0] = ((h >> 17) & 0xFFFF).to(torch.int32).to(torch.int16)
    return I, L


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=65536)
    ap.add_argument("--tile", type=int, default=8192)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--groups", default="intensity,moments,glcm")
    ap.add_argument("--sharded", action="store_true")
    ap.add_argument("--roll", type=int, default=None, help="rows to roll (default tile/2)")
    ap.add_argument("--phase", action="store_true", help="print k_roi_b phase clocks "
                    "(FXG_LIB pointing at a -DFXG_PHASE_TIMING build)")
    args = ap.parse_args()
    import torch
    import torch.distributed as dist

    import paper_2603_12016_b200 as fx
    from tools import synth
    from paper_2603_12016_b200 import shard
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if args.sharded:
        dist.init_process_group("nccl", device_id=dev)
    groups = args.groups.split(",")
    p = fx.resolve_profile("default")
    mask = fx.resolve_groups(groups)
    ncols = len(fx.feature_columns(mask, p))
    S, T = args.size, args.tile
    t0 = time.time()
    tile, rs = synth.packed_blob_mask_grid(T, 200000, 144, 1)
    per = int(tile.max())
    tile_lab = torch.from_numpy(tile.astype(np.int64)).to(dev)
    bands = shard.band_plan(S, world) if args.sharded else [(0, S)]
    y0, y1 = bands[rank]
    I, L = band_rasters(torch, dev, tile_lab, per, S, T, y0, y1, roll=args.roll)
    del tile_lab
    torch.cuda.synchronize()
    gen_s = time.time() - t0
    ctx = fx.Context(local)
    stream = torch.cuda.current_stream(dev)
    ctx.set_stream(stream.cuda_stream)
    if args.sharded:
        be = shard.DeviceBackend(ctx, mask, p)
        run = lambda: shard.featurize_band(be, dist, rank, world, I, L, y0, S, S)[0].numel()
    else:
        cap = per * (S // T) ** 2 + 16
        ol = torch.empty(cap, dtype=torch.int32, device=dev)
        ov = torch.empty((cap, ncols), dtype=torch.float64, device=dev)
        run = lambda: ctx.featurize_device(I.data_ptr(), L.data_ptr(), S, S, S, mask, p,
                                           ol.data_ptr(), ov.data_ptr(), cap)
    for _ in range(args.warmup):
        run()
    torch.cuda.synchronize()
    if args.sharded:
        dist.barrier()
    ctx.enable_timing(True)
    ctx.reset_kernel_times()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    from bench import ClockSampler
    n_own = 0
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            n_own = run()
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    kt = ctx.kernel_times()
    if args.phase:
        import ctypes as C
        from paper_2603_12016_b200 import fxg
        buf = (C.c_ulonglong * 16)()
        assert fxg.lib().fx_debug_phase_clocks(buf, 16, 1) == 0, "not a phase-timing build"
        names = ["words+scan", "pixels", "int hist/order", "edge+int out", "moments",
                 "glcm levels", "glcm angles"]
        tot = sum(buf[9:16])
        print("k_roi_b phases (thread 0, all steps):", ", ".join(
            f"{nm} {100 * buf[9 + k] / max(tot, 1):.1f}%" for k, nm in enumerate(names)), file=sys.stderr)
    n_all = n_own
    if args.sharded:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        c = torch.tensor([n_own], device=dev, dtype=torch.int64)
        dist.all_reduce(c)
        n_all = int(c.item())
    if rank == 0:
        alg = S * S * 4 + n_all * ncols * 8
        print(json.dumps({
            "metric": "megapixels/s", "unit": "MP/s", "value": S * S / 1e6 / (ms / 1e3),
            "rois_per_s": n_all / (ms / 1e3), "ms_per_step": ms, "steps": args.steps,
            "n_gpus": world, "scaling": "strong" if args.sharded else None,
            "config": {"workload": f"C5: {S}x{S} u16 whole slide, {n_all} blob ROIs (roi_size {rs}, "
                                   f"straddling 8192-row seams), groups {'+'.join(groups)}, "
                                   f"profile default",
                       "path": "row bands + NCCL table merge + halo (shard.py)" if args.sharded
                               else "one fx_featurize call",
                       "rasters_bytes": S * S * 4, "l2": "inputs >> L2"},
            "roofline": {"bound": "hbm", "algorithmic_bytes": alg,
                         "achieved_gbs": alg / (ms / 1e3) / 1e9},
            "kernels_ms_per_step_rank0": {k_: v[0] / args.steps for k_, v in sorted(kt.items())},
            "setup_s": gen_s, "clocks": clk.summary()}))
    ctx.close()
    if args.sharded:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
