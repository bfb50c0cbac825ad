#!/usr/bin/env python3
"""Per-feature-group throughput ({intensity, moments, glcm,
combined}) on the C2 image, and C3 (4096^2, 10k ROIs, GLCM ibsi-like): one JSON
line per (config, groups) with device MP/s and ROIs/s (device-resident inputs,
CUDA events), the per-kernel split, the call-level HBM fraction, nvidia-smi
clocks, and the reference CPU path (oracle/_ref, all host threads) on the same
image for the same groups.
usage: python tools/bench_groups.py [--steps K] [--no-ref]"""
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
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--no-ref", action="store_true")
    args = ap.parse_args()
    import torch

    import paper_2603_12016_b200 as fx
    from bench import ClockSampler, peaks
    from tools import synth
    hbm, _ = peaks()
    cases = []
    L2, _ = synth.packed_blob_mask_grid(8192, 400, 50000, 1)
    I2 = synth.uniform_u16(L2.shape, 0)
    for g in (["intensity"], ["moments"], ["glcm"], ["intensity", "moments"],
              ["intensity", "moments", "glcm"]):
        cases.append(("C2", I2, L2, g, "default"))
    L3, _ = synth.packed_blob_mask_grid(4096, 400, 10000, 1)
    I3 = synth.uniform_u16(L3.shape, 0)
    cases.append(("C3", I3, L3, ["glcm"], "ibsi-like"))
    ctx = fx.Context(0)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    for name, I, L, groups, prof in cases:
        h, w = L.shape
        p = fx.resolve_profile(prof)
        mask = fx.resolve_groups(groups)
        ncols = len(fx.feature_columns(mask, p))
        n = int(np.count_nonzero(np.bincount(L.ravel(), minlength=65536)[1:]))
        dI = torch.from_numpy(I.view(np.int16)).cuda()
        dL = torch.from_numpy(L.view(np.int16)).cuda()
        ol = torch.empty(n, dtype=torch.int32, device="cuda")
        ov = torch.empty((n, ncols), dtype=torch.float64, device="cuda")
        run = lambda: ctx.featurize_device(dI.data_ptr(), dL.data_ptr(), w, h, w, mask, p,
                                           ol.data_ptr(), ov.data_ptr(), n)
        for _ in range(3):
            run()
        ctx.enable_timing(True)
        ctx.timing_filter(None)
        ctx.reset_kernel_times()
        for _ in range(5):
            run()
        kt = ctx.kernel_times()
        ctx.enable_timing(False)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        with ClockSampler(0) as clk:
            e0.record(stream)
            for _ in range(args.steps):
                run()
            e1.record(stream)
            torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        call_bytes = h * w * 4 + n * ncols * 8
        line = {"config": name, "groups": groups, "profile": prof, "image": [h, w], "rois": n,
                "n_cols": ncols, "ms_per_step": round(ms, 4),
                "mp_per_s": round(h * w / 1e6 / (ms / 1e3), 1),
                "rois_per_s": round(n / (ms / 1e3), 1),
                "call_hbm_gbs": round(call_bytes / (ms / 1e3) / 1e9, 1),
                "call_hbm_frac": round(call_bytes / (ms / 1e3) / 1e9 / hbm, 4),
                "kernels_ms_per_step": {k: round(v[0] / 5, 4) for k, v in sorted(kt.items())},
                "clocks": clk.summary()}
        if not args.no_ref:
            from oracle import Reference, make_params
            ref = Reference()
            t0 = time.perf_counter()
            ref.featurize(I, L, groups, make_params(prof), threads=ref.max_threads())
            dt = time.perf_counter() - t0
            line["reference_cpu"] = {"mp_per_s": round(h * w / 1e6 / dt, 3),
                                     "rois_per_s": round(n / dt, 1), "threads": ref.max_threads(),
                                     "kind": "reference (oracle/_ref), one run"}
        print(json.dumps(line), flush=True)
        del dI, dL, ol, ov
    ctx.close()


if __name__ == "__main__":
    main()
