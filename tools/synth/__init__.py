"""BENCH / TEST TOOLING: synthetic inputs (not the product, not the oracle).

ctypes binding of tools/synth/_build/libfxsynth.so (fx_synth.cpp): the
reference's blob_mask_grid / siemens_star generators and mt19937_64 uniform
uint16 intensities, so bench.py and the tests build BASELINE.json's rasters on
the GPU box without the reference sources.  Checked pixel for pixel against the
reference's own generators in tests/test_synth.py.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "_build", "libfxsynth.so")
_lib = None


class SynthError(ValueError):
    pass


def _L():
    global _lib
    if _lib is None:
        if not os.path.exists(SO):
            subprocess.run(["make", "-s", "-C", os.path.dirname(os.path.dirname(HERE)), "synth"],
                           check=True)
        _lib = C.CDLL(SO)
    return _lib


def _check(rc, what):
    if rc:
        raise SynthError(f"{what}: invalid spec (code {rc})")


def _p(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint16))


def blob_mask_grid(image_size: int, roi_size: int, roi_count: int, seed: int = 1) -> np.ndarray:
    out = np.zeros((image_size, image_size), np.uint16)
    _check(_L().fxs_blob_mask_grid(image_size, roi_size, roi_count, C.c_uint64(seed), _p(out)),
           "blob_mask_grid")
    return out


def packed_blob_mask_grid(image_size: int, roi_size: int, roi_count: int, seed: int = 1):
    """blob_mask_grid, shrinking roi_size by 10% until it packs."""
    rs = roi_size
    while True:
        try:
            return blob_mask_grid(image_size, rs, roi_count, seed), rs
        except SynthError:
            rs = int(rs * 0.9)
            if rs < 1:
                raise


def siemens_star(size: int, spokes: int = 8) -> np.ndarray:
    out = np.zeros((size, size), np.uint16)
    _check(_L().fxs_siemens_star(size, spokes, _p(out)), "siemens_star")
    return out


def uniform_u16(shape, seed: int = 0) -> np.ndarray:
    out = np.zeros(shape, np.uint16)
    _check(_L().fxs_uniform_u16(C.c_uint64(seed), C.c_size_t(out.size), _p(out)), "uniform_u16")
    return out
