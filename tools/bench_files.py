#!/usr/bin/env python3
"""C4 end to end through the file path: PGM tiles on
disk -> featurex::run -> sorted %.10g CSV.

Tiles: 512 x 512, ~100 blob ROIs (packed_blob_mask_grid(512, 1000, 100, t % 16)),
uniform uint16 intensities (one seed per tile), written as 16-bit P5 files under
--dir (int/ and seg/, same basenames).  Times:
  ours : fx.run (C++ engine pipeline: parallel PGM decode into pinned buffers,
         fx_featurize_batch, parallel formatting) over all --tiles pairs, after a
         one-pair warm-up run (context creation, pinned allocation).
  ref  : the compiled reference's featurex::run (oracle/_ref, OpenMP, all host
         cores) over the first --ref-tiles pairs (a bounded sample).
The two CSVs are compared on the sample: labels exactly, values within 1e-6
relative (+1e-9 absolute: %.10g rounding of tiny values).
Prints one JSON line.
"""
from __future__ import annotations

import argparse
import csv
import json
import os
import shutil
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

TILE, ROIS, ROI_SIZE0, DISTINCT = 512, 100, 1000, 16


def write_tiles(d, n, first=0):
    import paper_2603_12016_b200 as fx
    from tools import synth
    labs = [synth.packed_blob_mask_grid(TILE, ROI_SIZE0, ROIS, s)[0] for s in range(DISTINCT)]
    for sub in ("int", "seg"):
        os.makedirs(os.path.join(d, sub), exist_ok=True)
    for t in range(first, first + n):
        name = f"t{t:05d}.pgm"
        I = np.random.default_rng(t).integers(0, 65536, (TILE, TILE), dtype=np.uint16)
        fx.write_pgm(os.path.join(d, "int", name), I, 65535)
        fx.write_pgm(os.path.join(d, "seg", name), labs[t % DISTINCT], 65535)
    return sum(int(np.count_nonzero(np.bincount(labs[t % DISTINCT].ravel())[1:]))
               for t in range(first, first + n))


def read_csv(path):
    with open(path) as f:
        r = csv.reader(f)
        head = next(r)
        rows = [row for row in r]
    keys = [(row[0], int(row[2])) for row in rows]
    vals = np.array([[float(x) for x in row[3:]] for row in rows]) if rows else np.zeros((0, len(head) - 3))
    return head, keys, vals


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tiles", type=int, default=2000)
    ap.add_argument("--ref-tiles", type=int, default=16)
    ap.add_argument("--groups", default="*ALL*")
    ap.add_argument("--dir", default="/tmp/fx_c4_files")
    ap.add_argument("--keep", action="store_true")
    args = ap.parse_args()
    import paper_2603_12016_b200 as fx
    groups = args.groups.split(",")
    shutil.rmtree(args.dir, ignore_errors=True)
    t0 = time.time()
    n_rois = write_tiles(args.dir, args.tiles)
    gen_s = time.time() - t0
    ncols = len(fx.feature_columns(groups, fx.resolve_profile("default")))
    out = os.path.join(args.dir, "ours.csv")
    # warm-up: one pair (context creation, kernel setup, pinned buffers)
    fx.run(os.path.join(args.dir, "int"), os.path.join(args.dir, "seg"), groups,
           output_path=out, pattern="t00000.pgm")
    s = fx.run(os.path.join(args.dir, "int"), os.path.join(args.dir, "seg"), groups,
               output_path=out)
    assert s.failed_pairs == 0 and s.images == args.tiles and s.rois == n_rois, (s.images, s.rois)
    csv_bytes = os.path.getsize(out)
    ours = {"seconds": s.elapsed_seconds, "tiles_per_s": args.tiles / s.elapsed_seconds,
            "MP_per_s": args.tiles * TILE * TILE / 1e6 / s.elapsed_seconds,
            "rois_per_s": n_rois / s.elapsed_seconds, "csv_MB": csv_bytes / 1e6}
    ref = None
    parity = None
    if args.ref_tiles > 0:
        try:
            from oracle import Reference
            R = Reference()
        except Exception as e:  # noqa: BLE001
            R = None
            ref = {"unavailable": str(e)}
        if R is not None:
            sub = os.path.join(args.dir, "sample")
            for kind in ("int", "seg"):
                os.makedirs(os.path.join(sub, kind), exist_ok=True)
                for t in range(args.ref_tiles):
                    os.link(os.path.join(args.dir, kind, f"t{t:05d}.pgm"),
                            os.path.join(sub, kind, f"t{t:05d}.pgm"))
            threads = R.max_threads()
            rout = os.path.join(sub, "ref.csv")
            rs = R.run(os.path.join(sub, "int"), os.path.join(sub, "seg"), groups, threads=threads,
                       parallel=True, output_path=rout)
            ref = {"seconds": rs.elapsed_seconds, "tiles": args.ref_tiles, "threads": threads,
                   "tiles_per_s": args.ref_tiles / rs.elapsed_seconds,
                   "MP_per_s": args.ref_tiles * TILE * TILE / 1e6 / rs.elapsed_seconds,
                   "rois_per_s": rs.rois / rs.elapsed_seconds}
            oout = os.path.join(sub, "ours.csv")
            fx.run(os.path.join(sub, "int"), os.path.join(sub, "seg"), groups, output_path=oout)
            h1, k1, v1 = read_csv(oout)
            h2, k2, v2 = read_csv(rout)
            same = h1 == h2 and k1 == k2
            if same:
                both_nan = np.isnan(v1) & np.isnan(v2)
                err = np.abs(v1 - v2)
                bound = 1e-6 * np.maximum(np.abs(v1), np.abs(v2)) + 1e-9
                ok = both_nan | (err <= bound)
                worst = {}
                for j in np.nonzero((~ok).any(axis=0))[0]:
                    r = err[:, j] / np.maximum(np.abs(v2[:, j]), 1e-300)
                    worst[h1[3 + j]] = {"cells": int((~ok[:, j]).sum()),
                                        "max_rel": float(np.nanmax(np.where(ok[:, j], 0, r))),
                                        "max_abs": float(np.nanmax(np.where(ok[:, j], 0, err[:, j])))}
                parity = {"rows": len(k1), "cells": int(ok.size), "cells_within_1e-6": int(ok.sum()),
                          "identical_text": open(oout).read() == open(rout).read(),
                          "outside": worst}
            else:
                parity = {"rows": len(k1), "header_or_labels_differ": True}
    print(json.dumps({
        "metric": "tiles/s (C4 files end to end: PGM decode -> device -> CSV)",
        "config": {"workload": f"C4 files: {args.tiles} x {TILE}x{TILE} 16-bit PGM pairs, "
                               f"{n_rois} ROIs, groups {'+'.join(groups)}, profile default",
                   "ncols": ncols, "generation_s": gen_s},
        "ours": ours, "reference": ref, "sample_parity": parity}))
    if not args.keep:
        shutil.rmtree(args.dir, ignore_errors=True)


if __name__ == "__main__":
    main()
