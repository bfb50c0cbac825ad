"""TEST INFRASTRUCTURE -- parity checkers, never the product.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this package.

* ``Oracle``    -- ctypes binding of oracle/_build/liboracle.so, the plain-C
                   restatement (oracle/fx_oracle.c) of the reference hot path.
* ``Reference`` -- ctypes binding of oracle/_ref/libfxref.so, the unmodified
                   reference sources (/root/reference/proj/src) compiled in
                   place with oracle/ref_shim.cpp.  Present whenever it was
                   built in the container (it travels to the GPU box as a
                   prebuilt .so); absent otherwise.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libfxref.so")

GROUP_BITS = {"intensity": 1, "shape": 2, "moments": 4, "glcm": 8, "glrlm": 16,
              "glszm": 32, "ngtdm": 64}
ALL_GROUPS = ["intensity", "shape", "moments", "glcm", "glrlm", "glszm", "ngtdm"]

PROFILES = {  # resolve_profile, reference engine.cpp:71-86
    "default": dict(ng=64, offset=1, angles=(0, 45, 90, 135), symmetric=True, histogram_bins=256),
    "performance": dict(ng=32, offset=1, angles=(0,), symmetric=False, histogram_bins=256),
    "ibsi-like": dict(ng=256, offset=1, angles=(0, 45, 90, 135), symmetric=True, histogram_bins=256),
}


class Params(C.Structure):
    _fields_ = [("ng", C.c_int), ("offset", C.c_int), ("n_angles", C.c_int),
                ("angles", C.c_int * 8), ("symmetric", C.c_int), ("histogram_bins", C.c_int)]


def make_params(profile="default", **over) -> Params:
    d = dict(PROFILES[profile])
    d.update(over)
    p = Params()
    p.ng, p.offset = int(d["ng"]), int(d["offset"])
    angles = list(d["angles"])
    p.n_angles = len(angles)
    for i, a in enumerate(angles):
        p.angles[i] = int(a)
    p.symmetric = 1 if d["symmetric"] else 0
    p.histogram_bins = int(d["histogram_bins"])
    return p


def group_mask(groups) -> int:
    m = 0
    for g in groups:
        if g == "*ALL*":
            m |= 127
        else:
            m |= GROUP_BITS[g]
    return m


def _u16(a):
    return np.ascontiguousarray(a, dtype=np.uint16)


def _ptr(a, t):
    return a.ctypes.data_as(C.POINTER(t))


def build_oracle():
    """Compile the C restatement if missing (gcc is in the image on both sides)."""
    if not os.path.exists(ORACLE_SO):
        subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"code {code}: {msg}")
        self.code = code


class Oracle:
    """The C restatement (fx_oracle.c)."""

    def __init__(self):
        build_oracle()
        L = C.CDLL(ORACLE_SO)
        self.L = L
        L.fxo_last_error.restype = C.c_char_p
        L.fxo_n_cols.argtypes = [C.c_uint, C.POINTER(Params)]

    def _check(self, rc):
        if rc:
            raise OracleError(rc, self.L.fxo_last_error().decode())

    def n_cols(self, groups, params):
        return self.L.fxo_n_cols(group_mask(groups), C.byref(params))

    def roi_table(self, labels):
        labels = _u16(labels)
        h, w = labels.shape
        cap = 65535
        ol = np.zeros(cap, np.uint32)
        oc = np.zeros(cap, np.uint64)
        ob = np.zeros((cap, 4), np.uint32)
        n = C.c_size_t()
        self._check(self.L.fxo_roi_table(_ptr(labels, C.c_uint16), w, h, _ptr(ol, C.c_uint32),
                                         _ptr(oc, C.c_uint64), _ptr(ob, C.c_uint32),
                                         C.c_size_t(cap), C.byref(n)))
        k = n.value
        return ol[:k].copy(), oc[:k].copy(), ob[:k].copy()

    def featurize(self, intensity, labels, groups, params):
        intensity, labels = _u16(intensity), _u16(labels)
        h, w = labels.shape
        nc = self.n_cols(groups, params)
        cap = int(np.count_nonzero(np.bincount(labels.ravel(), minlength=65536)[1:]))
        ol = np.zeros(max(cap, 1), np.uint32)
        ov = np.zeros((max(cap, 1), nc), np.float64)
        n, ncol = C.c_size_t(), C.c_int()
        self._check(self.L.fxo_featurize(_ptr(intensity, C.c_uint16), _ptr(labels, C.c_uint16),
                                         w, h, C.c_uint(group_mask(groups)), C.byref(params),
                                         _ptr(ol, C.c_uint32), _ptr(ov, C.c_double),
                                         C.c_size_t(cap), C.byref(n), C.byref(ncol)))
        return ol[:n.value], ov[:n.value]

    def roi_features(self, xs, ys, vs, groups, params):
        xs = np.ascontiguousarray(xs, np.uint32)
        ys = np.ascontiguousarray(ys, np.uint32)
        vs = _u16(vs)
        nc = self.n_cols(groups, params)
        out = np.zeros(nc, np.float64)
        ncol = C.c_int()
        self._check(self.L.fxo_roi_features(_ptr(xs, C.c_uint32), _ptr(ys, C.c_uint32),
                                            _ptr(vs, C.c_uint16), C.c_size_t(len(xs)),
                                            C.c_uint(group_mask(groups)), C.byref(params),
                                            _ptr(out, C.c_double), C.c_size_t(nc),
                                            C.byref(ncol)))
        return out

    def trace_contour(self, xs, ys):
        xs = np.ascontiguousarray(xs, np.uint32)
        ys = np.ascontiguousarray(ys, np.uint32)
        cap = 16 * len(xs) + 64
        out = np.zeros(2 * cap, np.int32)
        n = C.c_size_t()
        self._check(self.L.fxo_trace_contour(_ptr(xs, C.c_uint32), _ptr(ys, C.c_uint32),
                                             C.c_size_t(len(xs)), _ptr(out, C.c_int32),
                                             C.c_size_t(cap), C.byref(n)))
        return out[: 2 * n.value].reshape(-1, 2)

    def glcm_counts(self, xs, ys, vs, ng, offset, angle, symmetric):
        xs = np.ascontiguousarray(xs, np.uint32)
        ys = np.ascontiguousarray(ys, np.uint32)
        vs = _u16(vs)
        counts = np.zeros(ng * ng, np.uint64)
        pairs = C.c_uint64()
        self._check(self.L.fxo_glcm_counts(_ptr(xs, C.c_uint32), _ptr(ys, C.c_uint32),
                                           _ptr(vs, C.c_uint16), C.c_size_t(len(xs)), ng, offset,
                                           angle, int(bool(symmetric)), _ptr(counts, C.c_uint64),
                                           C.byref(pairs)))
        return counts.reshape(ng, ng), pairs.value

    def intensity_hist(self, vs, bins):
        vs = _u16(vs)
        nb = max(2, bins)
        hist = np.zeros(nb, np.uint64)
        self._check(self.L.fxo_intensity_hist(_ptr(vs, C.c_uint16), C.c_size_t(len(vs)), bins,
                                              _ptr(hist, C.c_uint64)))
        return hist


class RunSummary(C.Structure):
    _fields_ = [("images", C.c_int), ("rois", C.c_uint64), ("rows", C.c_uint64),
                ("elapsed_seconds", C.c_double), ("failed_pairs", C.c_int)]


def reference_available() -> bool:
    return os.path.exists(REF_SO)


class Reference:
    """The unmodified reference library (oracle/_ref/libfxref.so)."""

    def __init__(self):
        if not reference_available():
            raise FileNotFoundError(REF_SO)
        L = C.CDLL(REF_SO)
        self.L = L
        L.fxref_last_error.restype = C.c_char_p

    def _check(self, rc):
        if rc:
            raise OracleError(rc, self.L.fxref_last_error().decode())

    def max_threads(self):
        return self.L.fxref_max_threads()

    def resolve_profile(self, name):
        p = Params()
        self._check(self.L.fxref_resolve_profile(name.encode(), C.byref(p)))
        return p

    def columns(self, groups, params):
        need, nc = C.c_size_t(), C.c_int()
        self._check(self.L.fxref_columns(",".join(groups).encode(), C.byref(params), None,
                                         C.c_size_t(0), C.byref(need), C.byref(nc)))
        buf = C.create_string_buffer(need.value)
        self._check(self.L.fxref_columns(",".join(groups).encode(), C.byref(params), buf,
                                         C.c_size_t(need.value), C.byref(need), C.byref(nc)))
        s = buf.value.decode()
        return s.split("\n") if s else []

    def featurize(self, intensity, labels, groups, params, threads=1):
        intensity, labels = _u16(intensity), _u16(labels)
        h, w = labels.shape
        nc = len(self.columns(groups, params))
        cap = int(np.count_nonzero(np.bincount(labels.ravel(), minlength=65536)[1:]))
        ol = np.zeros(max(cap, 1), np.uint32)
        ov = np.zeros((max(cap, 1), nc), np.float64)
        n, ncol = C.c_size_t(), C.c_int()
        self._check(self.L.fxref_featurize(_ptr(intensity, C.c_uint16), _ptr(labels, C.c_uint16),
                                           w, h, ",".join(groups).encode(), C.byref(params),
                                           int(threads), _ptr(ol, C.c_uint32),
                                           _ptr(ov, C.c_double), C.c_size_t(cap), C.byref(n),
                                           C.byref(ncol)))
        return ol[:n.value], ov[:n.value]

    def roi_table(self, intensity, labels, rows_per_tile=256):
        intensity, labels = _u16(intensity), _u16(labels)
        h, w = labels.shape
        cap = 65535
        ol = np.zeros(cap, np.uint32)
        oc = np.zeros(cap, np.uint64)
        ob = np.zeros((cap, 4), np.uint32)
        n = C.c_size_t()
        self._check(self.L.fxref_roi_table(_ptr(intensity, C.c_uint16), _ptr(labels, C.c_uint16),
                                           w, h, rows_per_tile, _ptr(ol, C.c_uint32),
                                           _ptr(oc, C.c_uint64), _ptr(ob, C.c_uint32),
                                           C.c_size_t(cap), C.byref(n)))
        k = n.value
        return ol[:k].copy(), oc[:k].copy(), ob[:k].copy()

    def roi_features(self, xs, ys, vs, groups, params):
        xs = np.ascontiguousarray(xs, np.uint32)
        ys = np.ascontiguousarray(ys, np.uint32)
        vs = _u16(vs)
        cap = 2048
        out = np.zeros(cap, np.float64)
        ncol = C.c_int()
        self._check(self.L.fxref_roi_features(_ptr(xs, C.c_uint32), _ptr(ys, C.c_uint32),
                                              _ptr(vs, C.c_uint16), C.c_size_t(len(xs)),
                                              ",".join(groups).encode(), C.byref(params),
                                              _ptr(out, C.c_double), C.c_size_t(cap),
                                              C.byref(ncol)))
        return out[: ncol.value].copy()

    def trace_contour(self, xs, ys):
        xs = np.ascontiguousarray(xs, np.uint32)
        ys = np.ascontiguousarray(ys, np.uint32)
        cap = 16 * len(xs) + 64
        out = np.zeros(2 * cap, np.int32)
        n = C.c_size_t()
        self._check(self.L.fxref_trace_contour(_ptr(xs, C.c_uint32), _ptr(ys, C.c_uint32),
                                               C.c_size_t(len(xs)), _ptr(out, C.c_int32),
                                               C.c_size_t(cap), C.byref(n)))
        return out[: 2 * n.value].reshape(-1, 2)

    def glcm(self, xs, ys, vs, ng, offset, angle, symmetric):
        xs = np.ascontiguousarray(xs, np.uint32)
        ys = np.ascontiguousarray(ys, np.uint32)
        vs = _u16(vs)
        p = np.zeros(ng * ng, np.float64)
        pairs = C.c_uint64()
        self._check(self.L.fxref_glcm(_ptr(xs, C.c_uint32), _ptr(ys, C.c_uint32),
                                      _ptr(vs, C.c_uint16), C.c_size_t(len(xs)), ng, offset, angle,
                                      int(bool(symmetric)), _ptr(p, C.c_double), C.byref(pairs)))
        return p.reshape(ng, ng), pairs.value

    def blob_mask_grid(self, image_size, roi_size, roi_count, seed):
        out = np.zeros((image_size, image_size), np.uint16)
        self._check(self.L.fxref_blob_mask_grid(image_size, roi_size, roi_count,
                                                C.c_uint64(seed), _ptr(out, C.c_uint16)))
        return out

    def siemens_star(self, size, spokes=8):
        out = np.zeros((size, size), np.uint16)
        self._check(self.L.fxref_siemens_star(size, spokes, _ptr(out, C.c_uint16)))
        return out

    def run(self, intensity_dir, mask_dir, groups, profile="default", threads=1,
            parallel=True, output_path="out.csv", pattern="*.pgm"):
        s = RunSummary()
        self._check(self.L.fxref_run(str(intensity_dir).encode(), str(mask_dir).encode(),
                                     pattern.encode(), ",".join(groups).encode(),
                                     profile.encode(), int(threads), int(bool(parallel)),
                                     str(output_path).encode(), C.byref(s)))
        return s
