#!/usr/bin/env python3
"""C5 workload (BASELINE.json configs[4]) on one GPU: a 65536 x 65536 uint16
whole-slide image with large blob ROIs, featurized in one fx_featurize call on
device-resident rasters (17.2 GB; the band-sharded multi-GPU path is
paper_2603_12016_b200/shard.py).

Labels: blob_mask_grid(8192, 200000, 144, seed 1) (12 x 12 blobs of ~2e5 px),
replicated 8 x 8 with distinct label ranges (9216 ROIs), then rolled down by 4096
rows so blobs straddle every 8192-row band seam (the wrapped top/bottom blobs
become two-component ROIs).  Intensities: uniform uint16 drawn on the device.
Prints one JSON line.
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=65536)
    ap.add_argument("--tile", type=int, default=8192)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--groups", default="intensity,moments,glcm")
    args = ap.parse_args()
    import torch

    import paper_2603_12016_b200 as fx
    groups = args.groups.split(",")
    p = fx.resolve_profile("default")
    mask = fx.resolve_groups(groups)
    ncols = len(fx.feature_columns(mask, p))
    S, T = args.size, args.tile
    k = S // T
    t0 = time.time()
    tile, rs = fx.packed_blob_mask_grid(T, 200000, 144, 1)
    per = int(tile.max())
    dev = torch.device("cuda", 0)
    tl = torch.from_numpy(tile.astype(np.int32)).to(dev)
    L = torch.empty((S, S), dtype=torch.int16, device=dev)
    for by in range(k):
        for bx in range(k):
            off = (by * k + bx) * per
            t = torch.where(tl > 0, tl + off, torch.zeros_like(tl))
            L[by * T:(by + 1) * T, bx * T:(bx + 1) * T] = t.to(torch.int32).to(torch.int16)
    del tl
    L = torch.roll(L, shifts=T // 2, dims=0).contiguous()
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    I = torch.randint(-32768, 32768, (S, S), dtype=torch.int16, device=dev, generator=g)
    n_rois = per * k * k
    cap = n_rois + 16
    ol = torch.empty(cap, dtype=torch.int32, device=dev)
    ov = torch.empty((cap, ncols), dtype=torch.float64, device=dev)
    torch.cuda.synchronize()
    gen_s = time.time() - t0
    ctx = fx.Context(0)
    stream = torch.cuda.current_stream(dev)
    ctx.set_stream(stream.cuda_stream)
    run = lambda: ctx.featurize_device(I.data_ptr(), L.data_ptr(), S, S, S, mask, p,
                                       ol.data_ptr(), ov.data_ptr(), cap)
    for _ in range(args.warmup):
        n = run()
    torch.cuda.synchronize()
    ctx.enable_timing(True)
    ctx.reset_kernel_times()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        n = run()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    kt = ctx.kernel_times()
    mp = S * S / 1e6
    fg = float((L != 0).float().mean().item())
    alg = S * S * 4 + n * ncols * 8
    print(json.dumps({
        "metric": "megapixels/s", "unit": "MP/s", "value": mp / (ms / 1e3),
        "rois_per_s": n / (ms / 1e3), "ms_per_step": ms, "steps": args.steps, "n_gpus": 1,
        "config": {"workload": f"C5 on one GPU: {S}x{S} u16 whole slide, {n} blob ROIs "
                               f"(roi_size {rs}, {fg:.1%} fg, straddling 8192-row seams), "
                               f"groups {'+'.join(groups)}, profile default",
                   "rasters_bytes": S * S * 4, "l2": "inputs >> L2"},
        "roofline": {"bound": "hbm", "algorithmic_bytes": alg,
                     "achieved_gbs": alg / (ms / 1e3) / 1e9},
        "kernels_ms_per_step": {k_: v[0] / args.steps for k_, v in sorted(kt.items())},
        "setup_s": gen_s}))
    ctx.close()


if __name__ == "__main__":
    main()
