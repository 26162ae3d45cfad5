"""ctypes binding of include/dmsgm_klt.h: GPU estimation of the per-frame homographies
(App. F).  Argument marshalling only -- every
step runs in libdmsgm.so's kernels; there is no CPU fallback.  Names follow the header.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, fields

from .dmsgm import DMSGM_OK, DmsgmError, _check_tensor, _ptr, _stream_handle, lib

KLT_EXPORTS = ("dmsgm_klt_create", "dmsgm_klt_estimate", "dmsgm_klt_estimate_seq", "dmsgm_klt_seq_reset",
               "dmsgm_klt_corners", "dmsgm_klt_track",
               "dmsgm_klt_ransac", "dmsgm_klt_get_status", "dmsgm_klt_levels",
               "dmsgm_klt_kernels_per_estimate", "dmsgm_klt_last_error", "dmsgm_klt_destroy")


class dmsgm_klt_params(ctypes.Structure):
    _fields_ = [("num_streams", ctypes.c_int), ("max_corners", ctypes.c_int), ("quality", ctypes.c_double),
                ("min_distance", ctypes.c_double), ("win", ctypes.c_int), ("max_level", ctypes.c_int),
                ("max_iters", ctypes.c_int), ("eps", ctypes.c_float), ("min_eig", ctypes.c_float),
                ("ransac_iters", ctypes.c_int), ("ransac_thresh", ctypes.c_double),
                ("seed", ctypes.c_ulonglong)]


@dataclass
class KltParams:
    """dmsgm_klt_params with the defaults of DESIGN.md R38-R42 (App. F's Size(20,20), 5)."""
    num_streams: int = 1
    max_corners: int = 400
    quality: float = 0.01
    min_distance: float = 10.0
    win: int = 20
    max_level: int = 5
    max_iters: int = 30
    eps: float = 0.01
    min_eig: float = 1e-3
    ransac_iters: int = 500
    ransac_thresh: float = 3.0
    seed: int = 42

    def to_c(self) -> dmsgm_klt_params:
        return dmsgm_klt_params(*[getattr(self, f.name) for f in fields(self)])


def _setup(L):
    if getattr(L, "_klt_ready", False):
        return L
    P, i32, sz = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t
    L.dmsgm_klt_create.argtypes = [i32, i32, ctypes.POINTER(dmsgm_klt_params), i32, ctypes.POINTER(P)]
    L.dmsgm_klt_estimate.argtypes = [P, P, sz, P, sz, P, P, P]
    L.dmsgm_klt_estimate_seq.argtypes = [P, P, sz, P, sz, P, P, P]
    L.dmsgm_klt_seq_reset.argtypes = [P]
    L.dmsgm_klt_corners.argtypes = [P, P, sz, P, P, P]
    L.dmsgm_klt_track.argtypes = [P, P, sz, P, sz, P, P, P, P, P]
    L.dmsgm_klt_ransac.argtypes = [P, P, P, P, P, P, P, P, P]
    L.dmsgm_klt_get_status.argtypes = [P, ctypes.POINTER(ctypes.c_uint)]
    L.dmsgm_klt_levels.argtypes = [P]
    L.dmsgm_klt_kernels_per_estimate.argtypes = [P]
    L.dmsgm_klt_last_error.argtypes = [P]
    L.dmsgm_klt_last_error.restype = ctypes.c_char_p
    L.dmsgm_klt_destroy.argtypes = [P]
    L.dmsgm_klt_destroy.restype = None
    L._klt_ready = True
    return L


class Klt:
    """One dmsgm_klt_ctx: S streams of width x height frames on `device`."""

    def __init__(self, width: int, height: int, params: KltParams, device: int = 0):
        self._lib = _setup(lib())
        self.width, self.height, self.params, self.device = width, height, params, device
        h = ctypes.c_void_p()
        cp = params.to_c()
        rc = self._lib.dmsgm_klt_create(width, height, ctypes.byref(cp), device, ctypes.byref(h))
        if rc != DMSGM_OK:
            raise DmsgmError(rc, self._lib.dmsgm_klt_last_error(None).decode())
        self._h = h
        self.levels = self._lib.dmsgm_klt_levels(h)
        self.kernels_per_estimate = self._lib.dmsgm_klt_kernels_per_estimate(h)

    def _check(self, rc):
        if rc != DMSGM_OK:
            raise DmsgmError(rc, self._lib.dmsgm_klt_last_error(self._h).decode())

    def _frames(self, name, t):
        S = self.params.num_streams
        _check_tensor(name, t, (S, self.height, self.width), "uint8", self.device, self.height)

    def close(self):
        if getattr(self, "_h", None):
            self._lib.dmsgm_klt_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def estimate(self, prev, nxt, H_out, ok_out=None, stream=None):
        """prev / next: uint8 CUDA [S][H][W]; H_out f64 [S][9] (frame t -> t-1); ok_out int32 [S]."""
        S = self.params.num_streams
        self._frames("prev", prev)
        self._frames("next", nxt)
        _check_tensor("H_out", H_out, (S, 9), "float64", self.device)
        if ok_out is not None:
            _check_tensor("ok_out", ok_out, (S,), "int32", self.device)
        self._check(self._lib.dmsgm_klt_estimate(self._h, _ptr(prev), prev.stride(-2), _ptr(nxt), nxt.stride(-2),
                                                 _ptr(H_out), _ptr(ok_out), _stream_handle(stream)))

    def estimate_seq(self, prev, nxt, H_out, ok_out=None, stream=None):
        """estimate() for consecutive pairs of a video: reuses the corners and pyramid of `prev`
        when it is the buffer passed as `nxt` to the previous call (its content unchanged --
        the caller's guarantee; seq_reset() otherwise), include/dmsgm_klt.h."""
        S = self.params.num_streams
        self._frames("prev", prev)
        self._frames("next", nxt)
        _check_tensor("H_out", H_out, (S, 9), "float64", self.device)
        if ok_out is not None:
            _check_tensor("ok_out", ok_out, (S,), "int32", self.device)
        self._check(self._lib.dmsgm_klt_estimate_seq(self._h, _ptr(prev), prev.stride(-2), _ptr(nxt), nxt.stride(-2),
                                                     _ptr(H_out), _ptr(ok_out), _stream_handle(stream)))

    def seq_reset(self):
        self._check(self._lib.dmsgm_klt_seq_reset(self._h))

    def corners(self, frames, corners_out, counts_out, stream=None):
        S, M = self.params.num_streams, self.params.max_corners
        self._frames("frames", frames)
        _check_tensor("corners_out", corners_out, (S, M, 2), "int32", self.device)
        _check_tensor("counts_out", counts_out, (S,), "int32", self.device)
        self._check(self._lib.dmsgm_klt_corners(self._h, _ptr(frames), frames.stride(-2), _ptr(corners_out),
                                                _ptr(counts_out), _stream_handle(stream)))

    def track(self, prev, nxt, corners, counts, tracked_out, status_out, stream=None):
        S, M = self.params.num_streams, self.params.max_corners
        self._frames("prev", prev)
        self._frames("next", nxt)
        _check_tensor("corners", corners, (S, M, 2), "int32", self.device)
        _check_tensor("counts", counts, (S,), "int32", self.device)
        _check_tensor("tracked_out", tracked_out, (S, M, 2), "float32", self.device)
        _check_tensor("status_out", status_out, (S, M), "uint8", self.device)
        self._check(self._lib.dmsgm_klt_track(self._h, _ptr(prev), prev.stride(-2), _ptr(nxt), nxt.stride(-2),
                                              _ptr(corners), _ptr(counts), _ptr(tracked_out), _ptr(status_out),
                                              _stream_handle(stream)))

    def ransac(self, src, dst, counts, H_out, inliers_out=None, iter_counts_out=None, ok_out=None, stream=None):
        S, M = self.params.num_streams, self.params.max_corners
        _check_tensor("src", src, (S, M, 2), "float64", self.device)
        _check_tensor("dst", dst, (S, M, 2), "float64", self.device)
        _check_tensor("counts", counts, (S,), "int32", self.device)
        _check_tensor("H_out", H_out, (S, 9), "float64", self.device)
        if inliers_out is not None:
            _check_tensor("inliers_out", inliers_out, (S, M), "uint8", self.device)
        if iter_counts_out is not None:
            _check_tensor("iter_counts_out", iter_counts_out, (S, self.params.ransac_iters), "int32", self.device)
        if ok_out is not None:
            _check_tensor("ok_out", ok_out, (S,), "int32", self.device)
        self._check(self._lib.dmsgm_klt_ransac(self._h, _ptr(src), _ptr(dst), _ptr(counts), _ptr(H_out),
                                               _ptr(inliers_out), _ptr(iter_counts_out), _ptr(ok_out),
                                               _stream_handle(stream)))

    def get_status(self) -> int:
        v = ctypes.c_uint(0)
        self._check(self._lib.dmsgm_klt_get_status(self._h, ctypes.byref(v)))
        return v.value
