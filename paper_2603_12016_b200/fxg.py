"""ctypes binding of libfxg.so (the C ABI in include/fxg.h).

This is a thin host mirror of the reference engine API (engine.hpp:22-81) for
Python callers, tests and bench.py.  Every compute call goes to the sm_100a
kernels; there is no CPU fallback: a missing library or device raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FXG_LIB") or os.path.join(_HERE, "lib", "libfxg.so")

FX_OK = 0
ERRORS = {1: "ConfigError", 2: "UnknownProfile", 3: "PairingError", 4: "IoError",
          5: "FormatError", 6: "ZeroMassError", 7: "CudaError", 8: "OutOfMemory",
          9: "NcclError", 10: "CapacityError", 11: "ArgumentError", 12: "InternalError"}
MEM_HOST, MEM_DEVICE = 0, 1
GROUP_BITS = {"intensity": 1, "shape": 2, "moments": 4, "glcm": 8, "glrlm": 16, "glszm": 32,
              "ngtdm": 64}


class FxError(RuntimeError):
    """Error raised for a non-zero fx_status; .kind names the reference exception."""

    def __init__(self, code: int, msg: str):
        self.code = code
        self.kind = ERRORS.get(code, f"code{code}")
        super().__init__(f"{self.kind}: {msg}")


class TextureParams(C.Structure):
    _fields_ = [("ng", C.c_int), ("offset", C.c_int), ("n_angles", C.c_int),
                ("angles", C.c_int * 8), ("symmetric", C.c_int), ("histogram_bins", C.c_int)]

    def as_dict(self):
        return dict(ng=self.ng, offset=self.offset, angles=tuple(self.angles[: self.n_angles]),
                    symmetric=bool(self.symmetric), histogram_bins=self.histogram_bins)


class FxImage(C.Structure):
    _fields_ = [("intensity", C.c_void_p), ("labels", C.c_void_p), ("width", C.c_int),
                ("height", C.c_int), ("pitch", C.c_size_t), ("origin_x", C.c_int),
                ("origin_y", C.c_int), ("mem_kind", C.c_int)]


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise FxError(7, f"{LIB_PATH} missing -- run __graft_entry__.build() (no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        L.fx_last_error.restype = C.c_char_p
        L.fx_ctx_launch_count.restype = C.c_uint64
        L.fx_ctx_launch_count.argtypes = [C.c_void_p]
        for fn in ("fx_ctx_destroy", "fx_ctx_enable_timing", "fx_ctx_reset_kernel_times"):
            getattr(L, fn).argtypes = [C.c_void_p] + ([C.c_int] if fn == "fx_ctx_enable_timing" else [])
        L.fx_ctx_set_stream.argtypes = [C.c_void_p, C.c_void_p]
        L.fx_ctx_timing_filter.argtypes = [C.c_void_p, C.c_char_p]
        L.fx_multi_destroy.argtypes = [C.c_void_p]
        L.fx_multi_ctx.restype = C.c_void_p
        _lib = L
    return _lib


def _check(rc):
    if rc != FX_OK:
        raise FxError(rc, lib().fx_last_error().decode())


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


def resolve_profile(name: str) -> TextureParams:
    p = TextureParams()
    _check(lib().fx_resolve_profile(name.encode(), C.byref(p)))
    return p


def make_params(profile="default", **over) -> TextureParams:
    p = resolve_profile(profile)
    for k, v in over.items():
        if k == "angles":
            p.n_angles = len(v)
            for i, a in enumerate(v):
                p.angles[i] = int(a)
        elif k == "symmetric":
            p.symmetric = int(bool(v))
        else:
            setattr(p, k, int(v))
    return p


def resolve_groups(names) -> int:
    arr = (C.c_char_p * max(1, len(names)))(*[n.encode() for n in names])
    m = C.c_uint()
    _check(lib().fx_resolve_groups(arr, len(names), C.byref(m)))
    return m.value


def feature_columns(groups, params: TextureParams):
    mask = groups if isinstance(groups, int) else resolve_groups(list(groups))
    need, nc = C.c_size_t(), C.c_int()
    _check(lib().fx_columns(C.c_uint(mask), C.byref(params), None, C.c_size_t(0), C.byref(need),
                            C.byref(nc)))
    buf = C.create_string_buffer(need.value)
    _check(lib().fx_columns(C.c_uint(mask), C.byref(params), buf, C.c_size_t(need.value),
                            C.byref(need), C.byref(nc)))
    s = buf.value.decode()
    return s.split("\n") if s else []


class RunSummary(C.Structure):
    _fields_ = [("images", C.c_int), ("rois", C.c_uint64), ("rows", C.c_uint64),
                ("elapsed_seconds", C.c_double), ("failed_pairs", C.c_int)]


def run(intensity_dir, mask_dir, groups, profile="default", threads=1, parallel=True,
        output_path="out.csv", pattern="*.pgm", device=0) -> RunSummary:
    """featurex::run (engine.hpp:77) on PGM directories through the engine's
    batched device pipeline (fx_run); writes the sorted %.10g CSV."""
    s = RunSummary()
    _check(lib().fx_run(str(intensity_dir).encode(), str(mask_dir).encode(), pattern.encode(),
                        ",".join(groups).encode(), profile.encode(), int(threads),
                        int(bool(parallel)), int(device), str(output_path).encode(), C.byref(s)))
    return s


def write_pgm(path, samples: np.ndarray, maxval: int | None = None):
    """Binary PGM P5 (pgm.cpp:101-124): big-endian 16-bit samples when maxval > 255."""
    a = np.asarray(samples)
    mv = int(a.max()) if maxval is None else int(maxval)
    mv = max(mv, 1)
    body = a.astype(">u2").tobytes() if mv > 255 else a.astype(np.uint8).tobytes()
    with open(path, "wb") as f:
        f.write(b"P5\n%d %d\n%d\n" % (a.shape[1], a.shape[0], mv))
        f.write(body)


class Context:
    """One fx_ctx (device scratch + stream).  Not thread-safe."""

    def __init__(self, device: int = 0):
        self.h = C.c_void_p()
        _check(lib().fx_ctx_create(int(device), C.byref(self.h)))
        self.device = device

    def close(self):
        if self.h:
            lib().fx_ctx_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_handle: int | None):
        _check(lib().fx_ctx_set_stream(self.h, C.c_void_p(stream_handle or 0)))

    def set_band_rows(self, rows: int):
        """Row-band height of the host-raster path (0 auto, < 0 off); results are
        identical either way (fx_ctx_set_band_rows)."""
        _check(lib().fx_ctx_set_band_rows(self.h, int(rows)))

    def set_packing(self, on: bool):
        """Banded host rasters cross PCIe packed (label change points + labelled
        intensities) or raw; results are identical either way (fx_ctx_set_packing)."""
        _check(lib().fx_ctx_set_packing(self.h, 1 if on else 0))

    def last_transfer(self):
        """(h2d_bytes, d2h_bytes) of the last host-raster call (fx_ctx_last_transfer)."""
        a, b = C.c_uint64(), C.c_uint64()
        _check(lib().fx_ctx_last_transfer(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def launch_count(self) -> int:
        return int(lib().fx_ctx_launch_count(self.h))

    def enable_timing(self, on=True):
        _check(lib().fx_ctx_enable_timing(self.h, int(bool(on))))

    def timing_filter(self, kernel: str | None):
        _check(lib().fx_ctx_timing_filter(self.h, kernel.encode() if kernel else None))

    def reset_kernel_times(self):
        _check(lib().fx_ctx_reset_kernel_times(self.h))

    def kernel_times(self):
        n = C.c_int()
        ms = (C.c_double * 64)()
        cnt = (C.c_uint64 * 64)()
        buf = C.create_string_buffer(4096)
        _check(lib().fx_ctx_kernel_times(self.h, buf, C.c_size_t(4096), ms, cnt, 64, C.byref(n)))
        names = buf.value.decode().split("\n") if n.value else []
        return {nm: (ms[i], int(cnt[i])) for i, nm in enumerate(names)}

    # ---- the hot path -------------------------------------------------------
    def featurize(self, intensity, labels, groups=("intensity",), params=None, origin=(0, 0),
                  cap_rois=None):
        """Host numpy rasters -> (labels[n], table[n, ncols]) (engine.cpp:300-336)."""
        intensity = np.ascontiguousarray(intensity, dtype=np.uint16)
        labels = np.ascontiguousarray(labels, dtype=np.uint16)
        if intensity.shape != labels.shape:
            raise FxError(3, "image/mask dimension mismatch")
        h, w = labels.shape
        params = params or resolve_profile("default")
        mask = groups if isinstance(groups, int) else resolve_groups(list(groups))
        ncols = len(feature_columns(mask, params))
        if cap_rois is None:
            cap_rois = int(np.count_nonzero(np.bincount(labels.ravel(), minlength=65536)[1:]))
        out_l = np.zeros(max(cap_rois, 1), np.uint32)
        out_v = np.zeros((max(cap_rois, 1), max(ncols, 1)), np.float64)
        im = FxImage(intensity.ctypes.data, labels.ctypes.data, w, h, w, int(origin[0]),
                     int(origin[1]), MEM_HOST)
        n = C.c_size_t()
        _check(lib().fx_featurize(self.h, C.byref(im), C.c_uint(mask), C.byref(params),
                                  _p(out_l, C.c_uint32), _p(out_v, C.c_double),
                                  C.c_size_t(cap_rois), C.byref(n)))
        k = n.value
        return out_l[:k], out_v[:k, :ncols]

    def featurize_device(self, intensity_ptr: int, labels_ptr: int, width: int, height: int,
                         pitch: int, groups, params, out_labels_ptr: int, out_values_ptr: int,
                         cap_rois: int, origin=(0, 0)) -> int:
        """Device-resident rasters and outputs (raw CUDA pointers); returns n_rois."""
        mask = groups if isinstance(groups, int) else resolve_groups(list(groups))
        im = FxImage(intensity_ptr, labels_ptr, width, height, pitch, int(origin[0]),
                     int(origin[1]), MEM_DEVICE)
        n = C.c_size_t()
        _check(lib().fx_featurize(self.h, C.byref(im), C.c_uint(mask), C.byref(params),
                                  C.c_void_p(out_labels_ptr), C.c_void_p(out_values_ptr),
                                  C.c_size_t(cap_rois), C.byref(n)))
        return n.value

    def featurize_host_ptrs(self, intensity_ptr: int, labels_ptr: int, width: int, height: int,
                            groups, params, out_labels_ptr: int, out_values_ptr: int,
                            cap_rois: int) -> int:
        """Host (e.g. pinned) rasters/outputs by raw pointer: the end-to-end call."""
        mask = groups if isinstance(groups, int) else resolve_groups(list(groups))
        im = FxImage(intensity_ptr, labels_ptr, width, height, width, 0, 0, MEM_HOST)
        n = C.c_size_t()
        _check(lib().fx_featurize(self.h, C.byref(im), C.c_uint(mask), C.byref(params),
                                  C.c_void_p(out_labels_ptr), C.c_void_p(out_values_ptr),
                                  C.c_size_t(cap_rois), C.byref(n)))
        return n.value

    def featurize_batch(self, pairs, groups=("intensity",), params=None, origins=None,
                        cap_rois=None):
        """Host list of (intensity, labels) pairs -> list of (labels, table) per image,
        each identical to featurize() on that pair (fx_featurize_batch)."""
        params = params or resolve_profile("default")
        mask = groups if isinstance(groups, int) else resolve_groups(list(groups))
        ncols = len(feature_columns(mask, params))
        keep, ims = [], (FxImage * max(1, len(pairs)))()
        cap = 0
        for i, (I, L) in enumerate(pairs):
            I = np.ascontiguousarray(I, dtype=np.uint16)
            L = np.ascontiguousarray(L, dtype=np.uint16)
            if I.shape != L.shape:
                raise FxError(3, "image/mask dimension mismatch")
            keep.append((I, L))
            h, w = L.shape
            ox, oy = origins[i] if origins is not None else (0, 0)
            ims[i] = FxImage(I.ctypes.data, L.ctypes.data, w, h, w, int(ox), int(oy), MEM_HOST)
            if cap_rois is None:
                cap += int(np.count_nonzero(np.bincount(L.ravel(), minlength=65536)[1:]))
        cap = cap if cap_rois is None else cap_rois
        offs = self.featurize_batch_raw(ims, len(pairs), mask, params, None, None, cap,
                                        ncols=ncols)
        out_l, out_v, offs = offs
        return [(out_l[offs[i]:offs[i + 1]], out_v[offs[i]:offs[i + 1], :ncols])
                for i in range(len(pairs))]

    def featurize_batch_raw(self, images, n, groups, params, out_labels_ptr, out_values_ptr,
                            cap_rois, ncols=None):
        """images: ctypes FxImage array.  With out_*_ptr None, host numpy outputs are
        allocated and (labels, values, row_offsets) returned; otherwise the row
        offsets only (outputs already written through the pointers)."""
        mask = groups if isinstance(groups, int) else resolve_groups(list(groups))
        offs = np.zeros(n + 1, np.uint64)
        if out_labels_ptr is None:
            ncols = ncols if ncols is not None else len(feature_columns(mask, params))
            out_l = np.zeros(max(cap_rois, 1), np.uint32)
            out_v = np.zeros((max(cap_rois, 1), max(ncols, 1)), np.float64)
            lp, vp = _p(out_l, C.c_uint32), _p(out_v, C.c_double)
        else:
            lp, vp = C.c_void_p(out_labels_ptr), C.c_void_p(out_values_ptr)
        _check(lib().fx_featurize_batch(self.h, images, C.c_int(n), C.c_uint(mask),
                                        C.byref(params), lp, vp, C.c_size_t(cap_rois),
                                        _p(offs, C.c_size_t)))
        offs = offs.astype(np.int64)
        if out_labels_ptr is None:
            k = int(offs[n])
            return out_l[:k], out_v[:k], offs
        return offs

    def roi_features(self, xs, ys, vs, groups=("intensity",), params=None):
        """compute_roi_features on one cloud (engine.hpp:68-70)."""
        xs = np.ascontiguousarray(xs, np.uint32)
        ys = np.ascontiguousarray(ys, np.uint32)
        vs = np.ascontiguousarray(vs, np.uint16)
        params = params or resolve_profile("default")
        mask = groups if isinstance(groups, int) else resolve_groups(list(groups))
        ncols = len(feature_columns(mask, params))
        out = np.zeros(max(ncols, 1), np.float64)
        _check(lib().fx_roi_features(self.h, _p(xs, C.c_uint32), _p(ys, C.c_uint32),
                                     _p(vs, C.c_uint16), C.c_size_t(len(xs)), C.c_uint(mask),
                                     C.byref(params), _p(out, C.c_double), C.c_size_t(len(out))))
        return out[:ncols]

    def roi_features_batch(self, clouds, groups=("intensity",), params=None):
        """fx_roi_features_batch: clouds = [(xs, ys, vs), ...]; returns [n, n_cols]."""
        params = params or resolve_profile("default")
        mask = groups if isinstance(groups, int) else resolve_groups(list(groups))
        ncols = len(feature_columns(mask, params))
        sizes = [len(c[0]) for c in clouds]
        offs = np.zeros(len(clouds) + 1, dtype=np.uint64)
        offs[1:] = np.cumsum(sizes)
        cat = lambda i, t: (np.concatenate([np.asarray(c[i], t) for c in clouds])
                            if clouds else np.zeros(0, t))
        xs, ys, vs = cat(0, np.uint32), cat(1, np.uint32), cat(2, np.uint16)
        out = np.zeros((len(clouds), ncols))
        _check(lib().fx_roi_features_batch(self.h, _p(xs, C.c_uint32), _p(ys, C.c_uint32),
                                           _p(vs, C.c_uint16), _p(offs, C.c_size_t),
                                           C.c_size_t(len(clouds)), C.c_uint(mask), C.byref(params),
                                           _p(out, C.c_double), C.c_size_t(len(clouds))))
        return out

    def roi_table(self, intensity, labels, origin=(0, 0)):
        intensity = np.ascontiguousarray(intensity, dtype=np.uint16)
        labels = np.ascontiguousarray(labels, dtype=np.uint16)
        h, w = labels.shape
        cap = 65535
        ol = np.zeros(cap, np.uint32)
        oc = np.zeros(cap, np.uint64)
        ob = np.zeros((cap, 4), np.uint32)
        im = FxImage(intensity.ctypes.data, labels.ctypes.data, w, h, w, int(origin[0]),
                     int(origin[1]), MEM_HOST)
        n = C.c_size_t()
        _check(lib().fx_roi_table(self.h, C.byref(im), _p(ol, C.c_uint32), _p(oc, C.c_uint64),
                                  _p(ob, C.c_uint32), C.c_size_t(cap), C.byref(n)))
        k = n.value
        return ol[:k].copy(), oc[:k].copy(), ob[:k].copy()

    def debug_roi(self, intensity, labels, label, params=None):
        """Integer intermediates of one ROI: (hist, edge_xy, glcm[A,ng,ng], pairs[A])."""
        intensity = np.ascontiguousarray(intensity, dtype=np.uint16)
        labels = np.ascontiguousarray(labels, dtype=np.uint16)
        params = params or resolve_profile("default")
        h, w = labels.shape
        nb = max(2, params.histogram_bins)
        A, ng = params.n_angles, params.ng
        hist = np.zeros(nb, np.uint64)
        cap_edge = int((labels == label).sum()) + 8
        edge = np.zeros(2 * cap_edge, np.int32)
        glcm = np.zeros(A * ng * ng, np.uint32)
        pairs = np.zeros(A, np.uint64)
        ne = C.c_size_t()
        im = FxImage(intensity.ctypes.data, labels.ctypes.data, w, h, w, 0, 0, MEM_HOST)
        _check(lib().fx_debug_roi(self.h, C.byref(im), C.c_uint32(label), C.byref(params),
                                  _p(hist, C.c_uint64), _p(edge, C.c_int32), C.c_size_t(cap_edge),
                                  C.byref(ne), _p(glcm, C.c_uint32), _p(pairs, C.c_uint64)))
        return hist, edge[: 2 * ne.value].reshape(-1, 2), glcm.reshape(A, ng, ng), pairs


class Multi:
    """fx_multi: one context and host thread per listed device.
    A device may be listed more than once (several contexts share it)."""

    def __init__(self, devices):
        self.h = C.c_void_p()
        arr = (C.c_int * len(devices))(*devices)
        _check(lib().fx_multi_create(arr, len(devices), C.byref(self.h)))
        self.devices = list(devices)

    def close(self):
        if self.h:
            lib().fx_multi_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def featurize_batch(self, pairs, groups=("intensity",), params=None, cap_rois=None):
        """Host (intensity, labels) pairs -> [(labels, table)] per image, identical to
        Context.featurize_batch (fx_multi_featurize_batch)."""
        params = params or resolve_profile("default")
        mask = groups if isinstance(groups, int) else resolve_groups(list(groups))
        ncols = len(feature_columns(mask, params))
        keep, ims, cap = [], (FxImage * max(1, len(pairs)))(), 0
        for i, (I, L) in enumerate(pairs):
            I = np.ascontiguousarray(I, dtype=np.uint16)
            L = np.ascontiguousarray(L, dtype=np.uint16)
            if I.shape != L.shape:
                raise FxError(3, "image/mask dimension mismatch")
            keep.append((I, L))
            h, w = L.shape
            ims[i] = FxImage(I.ctypes.data, L.ctypes.data, w, h, w, 0, 0, MEM_HOST)
            if cap_rois is None:
                cap += int(np.count_nonzero(np.bincount(L.ravel(), minlength=65536)[1:]))
        cap = cap if cap_rois is None else cap_rois
        out_l = np.zeros(max(cap, 1), np.uint32)
        out_v = np.zeros((max(cap, 1), max(ncols, 1)), np.float64)
        offs = np.zeros(len(pairs) + 1, np.uint64)
        _check(lib().fx_multi_featurize_batch(self.h, ims, C.c_int(len(pairs)), C.c_uint(mask),
                                              C.byref(params), _p(out_l, C.c_uint32),
                                              _p(out_v, C.c_double), C.c_size_t(cap),
                                              _p(offs, C.c_size_t)))
        offs = offs.astype(np.int64)
        return [(out_l[offs[i]:offs[i + 1]], out_v[offs[i]:offs[i + 1], :ncols])
                for i in range(len(pairs))]

    def featurize_slide(self, intensity, labels, groups=("intensity",), params=None,
                        cap_rois=None, origin=(0, 0)):
        """One host image in row bands over the devices (fx_multi_featurize_slide);
        identical to Context.featurize on the whole image."""
        intensity = np.ascontiguousarray(intensity, dtype=np.uint16)
        labels = np.ascontiguousarray(labels, dtype=np.uint16)
        if intensity.shape != labels.shape:
            raise FxError(3, "image/mask dimension mismatch")
        h, w = labels.shape
        params = params or resolve_profile("default")
        mask = groups if isinstance(groups, int) else resolve_groups(list(groups))
        ncols = len(feature_columns(mask, params))
        if cap_rois is None:
            cap_rois = int(np.count_nonzero(np.bincount(labels.ravel(), minlength=65536)[1:]))
        out_l = np.zeros(max(cap_rois, 1), np.uint32)
        out_v = np.zeros((max(cap_rois, 1), max(ncols, 1)), np.float64)
        im = FxImage(intensity.ctypes.data, labels.ctypes.data, w, h, w, int(origin[0]),
                     int(origin[1]), MEM_HOST)
        n = C.c_size_t()
        _check(lib().fx_multi_featurize_slide(self.h, C.byref(im), C.c_uint(mask), C.byref(params),
                                              _p(out_l, C.c_uint32), _p(out_v, C.c_double),
                                              C.c_size_t(cap_rois), C.byref(n)))
        return out_l[:n.value], out_v[:n.value, :ncols]

