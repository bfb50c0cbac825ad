"""PCIe probe: pinned H2D / D2H / both directions at once for the C2 e2e sizes
(268 MB of rasters in, 57 MB of table out), and the C2 e2e call at several band
heights (fx_ctx_set_band_rows; 0 = auto, -1 = unbanded).  One JSON line."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def bw(fn, nbytes, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return nbytes * reps / (e0.elapsed_time(e1) / 1e3) / 1e9


def main():
    out = {}
    hin = torch.empty(268435456 // 2, dtype=torch.int16).pin_memory()
    din = torch.empty_like(hin, device="cuda")
    hout = torch.empty(57400000 // 8, dtype=torch.float64).pin_memory()
    dout = torch.empty_like(hout, device="cuda")
    out["h2d_gbs"] = round(bw(lambda: din.copy_(hin, non_blocking=True), hin.numel() * 2), 2)
    out["d2h_gbs"] = round(bw(lambda: hout.copy_(dout, non_blocking=True), hout.numel() * 8), 2)
    s2 = torch.cuda.Stream()

    def both():
        din.copy_(hin, non_blocking=True)
        with torch.cuda.stream(s2):
            hout.copy_(dout, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s2)
    out["h2d_plus_d2h_ms"] = round(1e3 * (hin.numel() * 2 + hout.numel() * 8) /
                                   bw(both, hin.numel() * 2 + hout.numel() * 8) / 1e9, 3)
    import bench
    import paper_2603_12016_b200 as fx
    I, L, _ = bench.workload(0)
    h, w = L.shape
    p = fx.resolve_profile(bench.PROFILE)
    mask = fx.resolve_groups(bench.GROUPS)
    ncols = len(fx.feature_columns(mask, p))
    n = bench.ROI_COUNT
    hI = torch.from_numpy(I.view(np.int16)).pin_memory()
    hL = torch.from_numpy(L.view(np.int16)).pin_memory()
    hv = torch.empty((n, ncols), dtype=torch.float64).pin_memory()
    hl = torch.empty(n, dtype=torch.int32).pin_memory()
    ctx = fx.Context(0)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    res = {}
    for rows in (-1, 0, 256, 512, 2048):
        ctx.set_band_rows(rows)
        run = lambda: ctx.featurize_host_ptrs(hI.data_ptr(), hL.data_ptr(), w, h, mask, p,
                                             hl.data_ptr(), hv.data_ptr(), n)
        for _ in range(2):
            run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            run()
        e1.record()
        torch.cuda.synchronize()
        res[str(rows)] = round(e0.elapsed_time(e1) / 10, 3)
    out["e2e_ms_by_band_rows"] = res
    print(json.dumps(out))


if __name__ == "__main__":
    main()
