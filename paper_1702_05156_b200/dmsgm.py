"""Thin ctypes binding of include/dmsgm.h -- argument marshalling only.

Every step of the path runs in libdmsgm.so (CUDA, sm_100a).  There is no CPU
fallback: importing this module raises if the library is missing.  Tensors are
PyTorch CUDA tensors used only as device memory; raw pointers and the current
CUDA stream are handed to the C ABI unchanged.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, fields

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
# DMSGM_LIB_PATH: load another build of the same C ABI (A/B timing of kernel versions)
LIB_PATH = os.environ.get("DMSGM_LIB_PATH") or os.path.join(_PKG, "libdmsgm.so")

DMSGM_OK = 0
DMSGM_EINVAL = -1
DMSGM_ENOMEM = -2
DMSGM_ECUDA = -3
DMSGM_ESTATE = -4
_ERRNAMES = {-1: "DMSGM_EINVAL", -2: "DMSGM_ENOMEM", -3: "DMSGM_ECUDA", -4: "DMSGM_ESTATE"}

# Every symbol include/dmsgm.h declares (checked by tests/test_abi.py).
EXPORTS = ("dmsgm_create", "dmsgm_step", "dmsgm_step_n", "dmsgm_step_host", "dmsgm_step_host_async", "dmsgm_reset",
           "dmsgm_get_state", "dmsgm_set_state", "dmsgm_is_initialised", "dmsgm_get_info",
           "dmsgm_last_error", "dmsgm_destroy", "dmsgm_version",
           "dmsgm_set_band", "dmsgm_get_buffers", "dmsgm_attach_peer", "dmsgm_get_ipc_handles",
           "dmsgm_attach_peer_ipc", "dmsgm_band_signal", "dmsgm_band_wait", "dmsgm_band_sync",
           "dmsgm_get_status", "dmsgm_band_halo_needed", "dmsgm_set_prefilter", "dmsgm_prefilter",
           "dmsgm_set_motion", "dmsgm_warp_frames", "dmsgm_set_mask_format")
DMSGM_MC_MODELS = 0
DMSGM_MC_FRAME = 1
DMSGM_MASK_BYTES = 0
DMSGM_MASK_BITS = 1
DMSGM_IPC_BYTES = 192


class DmsgmError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{_ERRNAMES.get(code, code)}: {msg}")
        self.code = code


class dmsgm_params(ctypes.Structure):
    _fields_ = [("theta_s", ctypes.c_float), ("theta_d", ctypes.c_float),
                ("var_init", ctypes.c_float), ("age_cap", ctypes.c_float),
                ("var_floor_match", ctypes.c_float), ("var_floor_classify", ctypes.c_float),
                ("decay_lambda", ctypes.c_float), ("decay_var_thresh", ctypes.c_float),
                ("num_streams", ctypes.c_int), ("update_rule", ctypes.c_int),
                ("classify_rule", ctypes.c_int)]


class dmsgm_info(ctypes.Structure):
    _fields_ = [("width", ctypes.c_int), ("height", ctypes.c_int), ("block", ctypes.c_int),
                ("blocks_x", ctypes.c_int), ("blocks_y", ctypes.c_int),
                ("num_streams", ctypes.c_int), ("kernels_per_step", ctypes.c_int),
                ("band_row0", ctypes.c_int), ("band_rows", ctypes.c_int), ("band_halo", ctypes.c_int),
                ("state_bytes", ctypes.c_size_t), ("algorithmic_bytes_per_frame", ctypes.c_double),
                ("kernel", ctypes.c_char * 64)]


class dmsgm_buffers(ctypes.Structure):
    _fields_ = [("state", ctypes.c_void_p * 2), ("flags", ctypes.c_void_p), ("parity", ctypes.c_int),
                ("steps", ctypes.c_uint), ("row_bytes", ctypes.c_size_t), ("stream_bytes", ctypes.c_size_t)]


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: build it with `python -m paper_1702_05156_b200.build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    P, i32, sz = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t
    lib.dmsgm_create.argtypes = [i32, i32, i32, ctypes.POINTER(dmsgm_params), i32, ctypes.POINTER(P)]
    lib.dmsgm_step.argtypes = [P, P, sz, P, P, sz, P]
    lib.dmsgm_step_n.argtypes = [P, i32, P, sz, P, P, sz, P]
    lib.dmsgm_step_host.argtypes = [P, P, sz, P, P, sz, P]
    lib.dmsgm_step_host_async.argtypes = [P, P, sz, P, P, sz, P]
    lib.dmsgm_reset.argtypes = [P, i32]
    lib.dmsgm_get_state.argtypes = [P, i32, P]
    lib.dmsgm_set_state.argtypes = [P, i32, P]
    lib.dmsgm_is_initialised.argtypes = [P, i32]
    lib.dmsgm_get_info.argtypes = [P, ctypes.POINTER(dmsgm_info)]
    lib.dmsgm_last_error.argtypes = [P]
    lib.dmsgm_last_error.restype = ctypes.c_char_p
    lib.dmsgm_destroy.argtypes = [P]
    lib.dmsgm_destroy.restype = None
    lib.dmsgm_set_band.argtypes = [P, i32, i32, i32]
    lib.dmsgm_get_buffers.argtypes = [P, ctypes.POINTER(dmsgm_buffers)]
    lib.dmsgm_attach_peer.argtypes = [P, i32, ctypes.POINTER(dmsgm_buffers)]
    lib.dmsgm_get_ipc_handles.argtypes = [P, P, sz]
    lib.dmsgm_attach_peer_ipc.argtypes = [P, i32, P, sz]
    lib.dmsgm_band_signal.argtypes = [P, P]
    lib.dmsgm_band_wait.argtypes = [P, P]
    lib.dmsgm_band_sync.argtypes = [P, P]
    lib.dmsgm_get_status.argtypes = [P, ctypes.POINTER(ctypes.c_uint)]
    lib.dmsgm_band_halo_needed.argtypes = [i32, i32, i32, P, i32, i32, i32, ctypes.POINTER(ctypes.c_int)]
    lib.dmsgm_set_prefilter.argtypes = [P, i32, ctypes.c_float, i32]
    lib.dmsgm_set_motion.argtypes = [P, i32]
    lib.dmsgm_set_mask_format.argtypes = [P, i32]
    lib.dmsgm_warp_frames.argtypes = [i32, i32, i32, P, sz, P, P, sz, P]
    lib.dmsgm_prefilter.argtypes = [i32, i32, i32, P, sz, P, sz, i32, ctypes.c_float, i32, P]
    lib.dmsgm_version.argtypes = []
    lib.dmsgm_version.restype = ctypes.c_char_p
    return lib


_lib = load_library()


def lib() -> ctypes.CDLL:
    return _lib


@dataclass
class Params:
    """dmsgm_params with the DESIGN.md defaults (R7, R15)."""
    theta_s: float = 4.0
    theta_d: float = 4.0
    var_init: float = 255.0
    age_cap: float = 30.0
    var_floor_match: float = 0.1
    var_floor_classify: float = 0.25
    decay_lambda: float = 0.001
    decay_var_thresh: float = 2500.0
    num_streams: int = 1
    update_rule: int = 0
    classify_rule: int = 0

    def to_c(self) -> dmsgm_params:
        return dmsgm_params(*[getattr(self, f.name) for f in fields(self)])


def _ptr(x) -> ctypes.c_void_p:
    """Raw pointer of a torch tensor / numpy array / int (no copies)."""
    if x is None:
        return ctypes.c_void_p(0)
    if isinstance(x, int):
        return ctypes.c_void_p(x)
    if isinstance(x, np.ndarray):
        return ctypes.c_void_p(x.ctypes.data)
    return ctypes.c_void_p(x.data_ptr())


def _stream_handle(stream) -> ctypes.c_void_p:
    if stream is None:
        import torch
        stream = torch.cuda.current_stream()
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    return ctypes.c_void_p(stream.cuda_stream)


def _row_pitch(t) -> int:
    """Row pitch in bytes of a [..., H, W] uint8 tensor/array (stride of dim -2)."""
    if isinstance(t, np.ndarray):
        return t.strides[-2]
    return t.stride(-2) * t.element_size()


def _strides_bytes(t):
    if isinstance(t, np.ndarray):
        return tuple(t.strides), t.dtype.itemsize
    return tuple(st * t.element_size() for st in t.stride()), t.element_size()


def _dtype_name(t) -> str:
    return str(t.dtype).replace("torch.", "")


def _check_tensor(name, t, shape, dtype, device, pitch_rows=None):
    """Argument marshalling guard for the C ABI: the library reads raw pointers with the
    [..][rows][pitch] / [..][9] layouts include/dmsgm.h states, so dtype, shape, device and
    the outer strides are checked here (ValueError) before a pointer is passed.  Raw
    integer pointers are passed through unchecked."""
    if isinstance(t, int):
        return
    if _dtype_name(t) != dtype:
        raise ValueError(f"{name}: dtype {_dtype_name(t)}, expected {dtype}")
    ok = tuple(t.shape) == tuple(shape)
    if pitch_rows is not None:                   # images: the last dim may be a padded pitch >= width
        ok = tuple(t.shape[:-1]) == tuple(shape[:-1]) and t.shape[-1] >= shape[-1]
    if not ok:
        raise ValueError(f"{name}: shape {tuple(t.shape)}, expected {tuple(shape)}"
                         f"{' (last dim >= width)' if pitch_rows is not None else ''}")
    if device == "cpu":
        if not isinstance(t, np.ndarray) and t.is_cuda:
            raise ValueError(f"{name}: expected host memory, got a CUDA tensor")
    else:
        if isinstance(t, np.ndarray) or not t.is_cuda:
            raise ValueError(f"{name}: expected a CUDA tensor on device {device}")
        if t.device.index != device:
            raise ValueError(f"{name}: on cuda:{t.device.index}, the context is on cuda:{device}")
    st, es = _strides_bytes(t)
    if st[-1] != es:
        raise ValueError(f"{name}: the last dimension must be contiguous")
    if pitch_rows is None:                      # homographies: dense [..][9] f64
        expect = es
        for d in range(len(shape) - 1, -1, -1):
            if shape[d] > 1 and st[d] != expect:
                raise ValueError(f"{name}: must be contiguous")
            expect *= shape[d]
        return
    pitch = st[-2]                               # images: [..][rows][pitch] per image, images dense
    expect = pitch * pitch_rows
    for d in range(len(shape) - 3, -1, -1):
        if shape[d] > 1 and st[d] != expect:
            raise ValueError(f"{name}: dimension {d} stride {st[d]} B, expected {expect} B "
                             f"(images of {pitch_rows} rows x {pitch} B must be consecutive)")
        expect *= shape[d]


class Dmsgm:
    """Python view of one dmsgm_ctx.  Names follow include/dmsgm.h."""

    def __init__(self, width: int, height: int, block: int, params: Params, device: int = 0):
        self._lib = _lib
        self.width, self.height, self.block = width, height, block
        self.params = params
        h = ctypes.c_void_p()
        cp = params.to_c()
        rc = self._lib.dmsgm_create(width, height, block, ctypes.byref(cp), device, ctypes.byref(h))
        if rc != DMSGM_OK:
            raise DmsgmError(rc, self._lib.dmsgm_last_error(None).decode())
        self._h = h
        self.device = device
        self.mask_format = DMSGM_MASK_BYTES
        self.info = self.get_info()

    # -- helpers -------------------------------------------------------------
    def _check_args(self, frames, homographies, masks, lead, device):
        rows = self.info.band_rows * self.block            # pixel rows of a (band) image
        S = self.info.num_streams
        _check_tensor("frames", frames, (*lead, S, rows, self.width), "uint8", device, rows)
        mw = (self.width + 7) // 8 if self.mask_format == DMSGM_MASK_BITS else self.width   # bytes per mask row
        _check_tensor("masks", masks, (*lead, S, rows, mw), "uint8", device, rows)
        _check_tensor("homographies", homographies, (*lead, S, 9), "float64", device)

    def _check(self, rc: int):
        if rc < 0:
            raise DmsgmError(rc, self._lib.dmsgm_last_error(self._h).decode())
        return rc

    @property
    def handle(self) -> ctypes.c_void_p:
        return self._h

    def close(self):
        if getattr(self, "_h", None):
            self._lib.dmsgm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- C ABI ---------------------------------------------------------------
    def step(self, frames, homographies, masks, stream=None):
        """frames/masks: uint8 CUDA [S][H][W] (row pitch from strides); homographies f64 [S][9]."""
        self._check_args(frames, homographies, masks, (), self.device)
        self._check(self._lib.dmsgm_step(self._h, _ptr(frames), _row_pitch(frames), _ptr(homographies),
                                         _ptr(masks), _row_pitch(masks), _stream_handle(stream)))

    def step_n(self, T: int, frames, homographies, masks, stream=None):
        """frames/masks: uint8 CUDA [T][S][H][W]; homographies f64 [T][S][9]."""
        self._check_args(frames, homographies, masks, (T,), self.device)
        self._check(self._lib.dmsgm_step_n(self._h, T, _ptr(frames), _row_pitch(frames), _ptr(homographies),
                                           _ptr(masks), _row_pitch(masks), _stream_handle(stream)))

    def step_host(self, frames, homographies, masks, stream=None):
        """HOST buffers (numpy or pinned CPU tensors); synchronous."""
        self._check_args(frames, homographies, masks, (), "cpu")
        self._check(self._lib.dmsgm_step_host(self._h, _ptr(frames), _row_pitch(frames), _ptr(homographies),
                                              _ptr(masks), _row_pitch(masks), _stream_handle(stream)))

    def step_host_async(self, frames, homographies, masks, stream=None):
        """HOST buffers (pinned); returns after enqueueing (see include/dmsgm.h)."""
        self._check_args(frames, homographies, masks, (), "cpu")
        self._check(self._lib.dmsgm_step_host_async(self._h, _ptr(frames), _row_pitch(frames), _ptr(homographies),
                                                    _ptr(masks), _row_pitch(masks), _stream_handle(stream)))

    def reset(self, stream: int = -1):
        self._check(self._lib.dmsgm_reset(self._h, stream))

    def get_state(self, stream: int) -> np.ndarray:
        out = np.empty((6, self.info.blocks_y, self.info.blocks_x), np.float32)
        self._check(self._lib.dmsgm_get_state(self._h, stream, _ptr(out)))
        return out

    def set_state(self, stream: int, state: np.ndarray):
        st = np.ascontiguousarray(state, np.float32)
        assert st.shape == (6, self.info.blocks_y, self.info.blocks_x), st.shape
        self._check(self._lib.dmsgm_set_state(self._h, stream, _ptr(st)))

    def is_initialised(self, stream: int) -> bool:
        return bool(self._check(self._lib.dmsgm_is_initialised(self._h, stream)))

    def get_info(self) -> dmsgm_info:
        info = dmsgm_info()
        self._check(self._lib.dmsgm_get_info(self._h, ctypes.byref(info)))
        return info

    # -- preprocessing (include/dmsgm.h) ---------------------
    def set_prefilter(self, gauss_size: int = 5, gauss_sigma: float = 1.0, median_radius: int = 1):
        self._check(self._lib.dmsgm_set_prefilter(self._h, gauss_size, gauss_sigma, median_radius))
        self.info = self.get_info()

    def set_mask_format(self, fmt: int):
        """DMSGM_MASK_BYTES (0, default: 0 / 255 per pixel) or DMSGM_MASK_BITS (1: one bit per
        pixel, LSB first, masks [S][H][>= ceil(W/8)] bytes); see include/dmsgm.h."""
        self._check(self._lib.dmsgm_set_mask_format(self._h, fmt))
        self.mask_format = fmt

    def set_motion(self, mode: int):
        """DMSGM_MC_MODELS (0, default) or DMSGM_MC_FRAME (1, App. F frame warp)."""
        self._check(self._lib.dmsgm_set_motion(self._h, mode))
        self.info = self.get_info()

    # -- row band (include/dmsgm.h) -------------------------------
    def set_band(self, row0: int, rows: int, halo: int):
        self._check(self._lib.dmsgm_set_band(self._h, row0, rows, halo))
        self.info = self.get_info()

    def get_buffers(self) -> dmsgm_buffers:
        b = dmsgm_buffers()
        self._check(self._lib.dmsgm_get_buffers(self._h, ctypes.byref(b)))
        return b

    def attach_peer(self, side: int, peer: "Dmsgm | dmsgm_buffers | None"):
        if peer is None:
            self._check(self._lib.dmsgm_attach_peer(self._h, side, None))
        else:
            b = peer.get_buffers() if isinstance(peer, Dmsgm) else peer
            self._check(self._lib.dmsgm_attach_peer(self._h, side, ctypes.byref(b)))
        self.info = self.get_info()

    def get_ipc_handles(self) -> bytes:
        buf = ctypes.create_string_buffer(DMSGM_IPC_BYTES)
        self._check(self._lib.dmsgm_get_ipc_handles(self._h, buf, DMSGM_IPC_BYTES))
        return buf.raw

    def attach_peer_ipc(self, side: int, handles: bytes):
        buf = ctypes.create_string_buffer(bytes(handles), len(handles))
        self._check(self._lib.dmsgm_attach_peer_ipc(self._h, side, buf, len(handles)))
        self.info = self.get_info()

    def band_signal(self, stream=None):
        self._check(self._lib.dmsgm_band_signal(self._h, _stream_handle(stream)))

    def band_wait(self, stream=None):
        self._check(self._lib.dmsgm_band_wait(self._h, _stream_handle(stream)))

    def band_sync(self, stream=None):
        self._check(self._lib.dmsgm_band_sync(self._h, _stream_handle(stream)))

    def get_status(self) -> int:
        v = ctypes.c_uint(0)
        self._check(self._lib.dmsgm_get_status(self._h, ctypes.byref(v)))
        return v.value


def prefilter(frames, out, gauss_size: int = 5, gauss_sigma: float = 1.0, median_radius: int = 1, stream=None):
    """Stand-alone preprocessing of uint8 CUDA frames [count][H][W] into `out` (same shape)."""
    count, H, W = frames.shape
    rc = _lib.dmsgm_prefilter(W, H, count, _ptr(frames), _row_pitch(frames), _ptr(out), _row_pitch(out),
                              gauss_size, gauss_sigma, median_radius, _stream_handle(stream))
    if rc != DMSGM_OK:
        raise DmsgmError(rc, "dmsgm_prefilter failed")


def warp_frames(frames, homographies, out, stream=None):
    """Stand-alone App. F frame warp of uint8 CUDA frames [count][H][W] into `out`."""
    count, H, W = frames.shape
    rc = _lib.dmsgm_warp_frames(W, H, count, _ptr(frames), _row_pitch(frames), _ptr(homographies), _ptr(out),
                                _row_pitch(out), _stream_handle(stream))
    if rc != DMSGM_OK:
        raise DmsgmError(rc, "dmsgm_warp_frames failed")


def band_halo_needed(width: int, height: int, block: int, homographies: np.ndarray, row0: int, rows: int) -> int:
    """Halo rows band [row0, row0+rows) needs for HOST homographies f64 [count][9]."""
    H = np.ascontiguousarray(homographies, np.float64).reshape(-1, 9)
    out = ctypes.c_int(0)
    rc = _lib.dmsgm_band_halo_needed(width, height, block, _ptr(H), H.shape[0], row0, rows, ctypes.byref(out))
    if rc != DMSGM_OK:
        raise DmsgmError(rc, "dmsgm_band_halo_needed: bad arguments")
    return out.value


def version() -> str:
    return _lib.dmsgm_version().decode()
