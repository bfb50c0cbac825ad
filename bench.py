#!/usr/bin/env python3
"""Benchmark of the per-ROI featurization hot path (BASELINE.json metric).

Workload (BASELINE.json configs[1], "C2"): one 8192x8192 uint16 intensity image
(uniform, std::mt19937_64(seed)() & 0xffff) + uint16 label mask of ~50k
disk-with-ears blobs (blob_mask_grid, seed 1, roi_size shrunk by 10% until it
packs), feature groups intensity + moments (default profile).

One step = one fx_featurize call over the whole image:
  value : device-resident inputs (HBM) -> feature table in HBM; CUDA events on the
          launching stream, K steps, max over ranks.  268 MB of rasters > 126 MB L2,
          so no explicit flush is needed between steps.
  e2e   : the same call through the C ABI with pinned HOST rasters and a HOST table
          (H2D of both rasters + D2H of labels/table inside the timed region).
N>1: one process per GPU (torchrun), each rank featurizes its own image (file
sharding, no data-path collective) -> weak scaling; value = all ranks' MP / max time.

--impl reference: the reference's own CPU implementation (oracle/_ref, compiled
from /root/reference sources) on all host cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

IMAGE = 8192
ROI_COUNT = 50000
ROI_SIZE0 = 400
GROUPS = ["intensity", "moments"]
PROFILE = "default"
METRIC = "megapixels/s"
UNIT = "MP/s"


def workload(seed_intensity: int):
    from tools import synth  # bench tooling (tools/synth), not the product library
    labels, roi_size = synth.packed_blob_mask_grid(IMAGE, ROI_SIZE0, ROI_COUNT, 1)
    intensity = synth.uniform_u16(labels.shape, seed_intensity)
    return intensity, labels, roi_size


def config_dict(roi_size, n_rois, fg_frac, n):
    return {"workload": f"C2: {IMAGE}x{IMAGE} uint16 intensity + uint16 labels, "
                        f"{n_rois} blob ROIs (roi_size {roi_size}, {fg_frac:.1%} fg), "
                        f"groups {'+'.join(GROUPS)}, profile {PROFILE}",
            "image": [IMAGE, IMAGE], "rois_per_image": int(n_rois), "groups": GROUPS,
            "profile": PROFILE, "images_per_step": n, "sharding": "one image per GPU",
            "l2": "inputs (268 MB) larger than L2 (126 MB); no flush"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled while the timed region runs."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # the timed region starts only once nvidia-smi is sampling: its start-up
            # (NVML init, slow on a fresh box) overlapping the timed launches once
            # cost ~10% of the step
            t0 = time.time()
            while not self.rows and time.time() - t0 < 5.0:
                time.sleep(0.02)
            time.sleep(0.1)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx = float(r[1])
                for k, nm in enumerate(names):
                    if r[3 + k].lower().startswith("active"):
                        reasons.add(nm)
            except (ValueError, IndexError):
                pass
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def profiled_traffic(kernel):
    """dram read+write bytes per launch from the committed ncu capture, or None."""
    import re
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f).get("bytes_per_launch", {})
    norm = {re.sub(r"<(\d+).*>", r"\1", k): v for k, v in d.items()}
    return norm.get(kernel)


def roi_classes(labels):
    """Per present label: pixel count and window class, by the rule the compaction
    applies on the device (fx_scan.cu roi_class: S0 w<=33, h<=40, n<=768; S1/S2
    w, h <= 64 split at n = 1024; else L).  Host-side, outside any timed region."""
    ys, xs = np.nonzero(labels)
    lab = labels[ys, xs].astype(np.int64)
    n = np.bincount(lab, minlength=65536)
    big = np.iinfo(np.int64).max
    x0 = np.full(65536, big); x1 = np.full(65536, -1)
    y0 = np.full(65536, big); y1 = np.full(65536, -1)
    np.minimum.at(x0, lab, xs); np.maximum.at(x1, lab, xs)
    np.minimum.at(y0, lab, ys); np.maximum.at(y1, lab, ys)
    present = np.nonzero(n[1:])[0] + 1
    n, w, h = n[present], (x1 - x0 + 1)[present], (y1 - y0 + 1)[present]
    cls = np.where((w <= 33) & (h <= 40) & (n <= 768), 0,
                   np.where((w <= 64) & (h <= 64), np.where(n <= 1024, 1, 2), 3))
    return n, cls


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def cpu_reference(intensity, labels, steps, warmup, threads=None):
    """Reference CPU path (oracle/_ref): accumulate + OpenMP compute_roi_features."""
    from oracle import Reference, make_params
    ref = Reference()
    threads = threads or ref.max_threads()
    p = make_params(PROFILE)
    times = []
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        rl, rv = ref.featurize(intensity, labels, GROUPS, p, threads=threads)
        dt = time.perf_counter() - t0
        if i >= warmup:
            times.append(dt)
    return times, threads, rl, rv


def reference_sample(intensity, labels, steps, warmup, budget_s=60.0, full_step_s=1.2):
    """Bounded per-step sample of the C2 image for the reference arm: the full
    image when (steps + warmup) full steps fit the budget (~1.1 s each on 16
    threads), else a band of whole rows sized to it (>= 512 rows).  Returns
    (intensity, labels, description)."""
    total = max(1, steps + warmup)
    frac = min(1.0, budget_s / (total * full_step_s))
    if frac >= 1.0:
        return intensity, labels, "full C2 image per step"
    rows = max(512, int(IMAGE * frac) // 256 * 256)
    return (np.ascontiguousarray(intensity[:rows]), np.ascontiguousarray(labels[:rows]),
            f"rows 0..{rows} of the C2 image per step ({rows}x{IMAGE}, labels cut at the band "
            f"edge); MP/s on the band's pixels")


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    intensity, labels, roi_size = workload(0)
    n_rois = int(np.count_nonzero(np.bincount(labels.ravel(), minlength=65536)[1:]))
    steps, warmup = max(1, args.steps), args.warmup
    I_s, L_s, sample = reference_sample(intensity, labels, steps, warmup)
    times, threads, rl, _ = cpu_reference(I_s, L_s, steps, warmup)
    nr = len(rl)
    t = float(np.sum(times))
    mp = L_s.shape[0] * L_s.shape[1] / 1e6
    value = mp * len(times) / t
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": UNIT,
            "n_gpus": world, "steps": len(times), "warmup": warmup,
            "ms_per_step": round(1e3 * t / len(times), 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(roi_size, n_rois, float((labels > 0).mean()), 1),
            "rois_per_s": round(nr * len(times) / t, 1),
            "cpu_baseline": {"value": round(value, 3), "unit": UNIT, "cores": threads,
                             "kind": "reference",
                             "sample": f"{sample} ({len(times)} steps, accumulate + OpenMP "
                                       f"compute_roi_features over ROIs, {threads} threads)"},
            "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def spot_check(intensity, labels, gl, gv, rl, rv, cols, sample=2000, seed=0):
    """tests/parity.py's comparator (bit-exact classes + tolerances with floors) on
    a random sample of ROIs of the benchmarked image; labels compared in full."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from parity import compare, floors
    if not np.array_equal(gl, rl):
        return {"ok": False, "rois": int(len(rl)), "violations": ["label list differs"]}
    pick = np.sort(np.random.default_rng(seed).choice(len(rl), min(sample, len(rl)),
                                                      replace=False))
    lab_pick = np.where(np.isin(labels, rl[pick]), labels, 0).astype(np.uint16)
    s = floors(cols, rv[pick], intensity, lab_pick, rl[pick])
    bad = compare(cols, gv[pick], rv[pick], s)
    return {"ok": not bad, "rois_compared": int(len(pick)), "rois": int(len(rl)),
            "violations": [f"{c} x{r:.3g} ({n} rows)" for c, r, n in bad[:8]]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return

    import torch
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    import paper_2603_12016_b200 as fx
    intensity, labels, roi_size = workload(rank)  # each rank: its own image (file shard)
    h, w = labels.shape
    n_rois = int(np.count_nonzero(np.bincount(labels.ravel(), minlength=65536)[1:]))
    params = fx.resolve_profile(PROFILE)
    gmask = fx.resolve_groups(GROUPS)
    ncols = len(fx.feature_columns(gmask, params))

    ctx = fx.Context(local_rank)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)

    # device-resident rasters and outputs
    d_img = torch.from_numpy(intensity.view(np.int16).reshape(-1)).cuda()
    d_lab = torch.from_numpy(labels.view(np.int16).reshape(-1)).cuda()
    d_out = torch.empty((n_rois, ncols), dtype=torch.float64, device="cuda")
    d_ol = torch.empty((n_rois,), dtype=torch.int32, device="cuda")

    def step_device():
        return ctx.featurize_device(d_img.data_ptr(), d_lab.data_ptr(), w, h, w, gmask, params,
                                    d_ol.data_ptr(), d_out.data_ptr(), n_rois)

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        assert step_device() == n_rois
    barrier()
    # breakdown pass (not the timed region): every kernel event-timed, to name the
    # dominant kernel and report the per-kernel split; each timing event between
    # launches costs ~3 us of device time, so the timed region below times only
    # the dominant kernel
    bd_steps = max(3, min(args.steps, 20))
    ctx.enable_timing(True)
    ctx.timing_filter(None)
    ctx.reset_kernel_times()
    for _ in range(bd_steps):
        step_device()
    barrier()
    kall = ctx.kernel_times()
    dom_name = max(kall.items(), key=lambda kv: kv[1][0])[0]
    # timed region: K steps, the dominant kernel's launches bracketed by events
    ctx.timing_filter(dom_name)
    ctx.reset_kernel_times()
    l0 = ctx.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            step_device()
        e1.record(stream)
        barrier()
    launches = ctx.launch_count() - l0
    ktimes = ctx.kernel_times()
    ctx.enable_timing(False)
    ctx.timing_filter(None)
    t_dev = max_over_ranks(e0.elapsed_time(e1) / 1e3)

    # end-to-end through the C ABI with pinned host buffers
    h_img = torch.from_numpy(intensity.view(np.int16)).pin_memory()
    h_lab = torch.from_numpy(labels.view(np.int16)).pin_memory()
    h_out = torch.empty((n_rois, ncols), dtype=torch.float64).pin_memory()
    h_ol = torch.empty((n_rois,), dtype=torch.int32).pin_memory()

    def step_e2e():
        return ctx.featurize_host_ptrs(h_img.data_ptr(), h_lab.data_ptr(), w, h, gmask, params,
                                       h_ol.data_ptr(), h_out.data_ptr(), n_rois)

    for _ in range(2):
        step_e2e()
    e2e_steps = max(3, min(args.steps, 20))
    barrier()
    e0.record(stream)
    for _ in range(e2e_steps):
        step_e2e()
    e1.record(stream)
    barrier()
    t_e2e = max_over_ranks(e0.elapsed_time(e1) / 1e3)
    assert int(h_ol[0]) >= 1
    h2d_b, d2h_b = ctx.last_transfer()
    # the same call with raw rows over PCIe (no host packing), for reference
    ctx.set_packing(False)
    step_e2e()
    raw_h2d, _ = ctx.last_transfer()
    barrier()
    e0.record(stream)
    for _ in range(e2e_steps):
        step_e2e()
    e1.record(stream)
    barrier()
    t_e2e_raw = max_over_ranks(e0.elapsed_time(e1) / 1e3)
    ctx.set_packing(True)

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return

    mp_step = h * w / 1e6
    value = world * mp_step * args.steps / t_dev
    e2e_value = world * mp_step * e2e_steps / t_e2e

    # roofline of the dominant kernel (largest share of device time).  Algorithmic
    # bytes are SURVEY.md 8(d)'s per-unit figures, independent of internal passes
    # (DESIGN.md section 5): the label scan reads the label raster once (W*H*2); a
    # per-ROI kernel reads its ROIs' member labels + intensities (n*4) and writes
    # their feature rows (n_cols*8).  The internal passes (compaction, the serial
    # passes over staged values) move no compulsory bytes and get no fraction.
    hbm, peak_src = peaks()
    dom_ms, dom_cnt = ktimes[dom_name]
    fg = int(np.count_nonzero(labels))
    n_px, cls = roi_classes(labels)
    per_roi = lambda c: int((n_px[cls == c] * 4).sum() + (cls == c).sum() * ncols * 8)
    algo_bytes = {"k_label_scan": h * w * 2, "k_roi_s0": per_roi(0), "k_roi_s1": per_roi(1),
                  "k_roi_s2": per_roi(2), "k_roi_b": per_roi(3)}
    per_launch_s = dom_ms / 1e3 / max(1, dom_cnt)
    achieved = algo_bytes.get(dom_name, 0) / per_launch_s / 1e9
    call_bytes = h * w * 4 + n_rois * ncols * 8
    call_gbs = call_bytes / (t_dev / args.steps) / 1e9
    kernels = {}
    for k, (ms, cnt) in sorted(kall.items(), key=lambda kv: -kv[1][0]):
        per = ms / 1e3 / max(1, cnt)
        ab = algo_bytes.get(k)
        kernels[k] = {"ms_per_step": round(ms / bd_steps, 4),
                      "share": round(ms / max(1e-12, sum(v[0] for v in kall.values())), 4),
                      "algorithmic_bytes": ab,
                      "gbs": round(ab / per / 1e9, 1) if ab else None,
                      "frac": round(ab / per / 1e9 / hbm, 4) if ab else None}
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * t_dev / args.steps, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(roi_size, n_rois, fg / (h * w), world),
        "rois_per_s": round(world * n_rois * args.steps / t_dev, 1),
        "featurize_hbm_gbs": round(call_gbs, 1),
        "e2e": {"value": round(e2e_value, 2), "unit": UNIT,
                "h2d_bytes_per_step": int(h2d_b), "d2h_bytes_per_step": int(d2h_b),
                "steps": e2e_steps,
                "path": "host rasters packed by host threads (label change points + "
                        "labelled intensities), unpacked on the device"
                        if h2d_b < 2 * h * w * 2 else "raw row bands",
                "raw_rows": {"value": round(world * mp_step * e2e_steps / t_e2e_raw, 2),
                             "h2d_bytes_per_step": int(raw_h2d)}},
        "gpu_launches": int(launches),
        "kernels": kernels,
        "kernels_note": f"per-kernel split from a separate {bd_steps}-step pass with every "
                        f"kernel event-timed; the timed region times only {dom_name}",
        "roofline": {"kernel": dom_name, "bound": "hbm", "achieved": round(achieved, 1),
                     "peak": hbm, "unit": "GB/s", "frac": round(achieved / hbm, 4),
                     "traffic": profiled_traffic(dom_name), "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": int(algo_bytes.get(dom_name, 0)),
                     "call": {"achieved": round(call_gbs, 1), "frac": round(call_gbs / hbm, 4),
                              "bytes": int(call_bytes),
                              "note": "whole fx_featurize call: W*H*4 + n_rois*n_cols*8 over "
                                      "ms_per_step"}},
        "clocks": clk.summary(),
    }
    if not args.no_cpu_baseline and world == 1:
        times, threads, rl, rv = cpu_reference(intensity, labels, 1, 0)
        line["cpu_baseline"] = {"value": round(mp_step / times[0], 3), "unit": UNIT,
                                "cores": threads, "kind": "reference",
                                "sample": "one full C2 image (in-memory accumulate + OpenMP "
                                          "compute_roi_features, oracle/_ref)"}
        # parity spot check of the benchmarked output (outside every timed region):
        # the device table of the last device step against the reference's table
        line["parity_spot_check"] = spot_check(
            intensity, labels, d_ol.cpu().numpy().view(np.uint32), d_out.cpu().numpy(),
            rl, rv, fx.feature_columns(gmask, params))
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
