"""TEST INFRASTRUCTURE ONLY -- ctypes wrapper for the plain C DMSGM oracle.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.  The product path
(paper_1702_05156_b200) never imports it and shares no code with it.

The oracle follows PAPER.md §2.2-2.4 (Eqs. 3-10) and App. E step by step; the
readings where the paper is silent are listed in DESIGN.md §2.  Parity status
of every function is recorded in DESIGN.md §5 ("pinned" unless stated).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "dmsgm_oracle.c")
_SRC2 = os.path.join(_HERE, "prefilter_oracle.c")
_SRC3 = os.path.join(_HERE, "warp_oracle.c")
_SRC4 = os.path.join(_HERE, "dmsgm_plain.c")
_HDR = os.path.join(_HERE, "dmsgm_oracle.h")
_HDR2 = os.path.join(_HERE, "oracle_ctx.h")
LIB_PATH = os.path.join(_HERE, "libdmsgm_oracle.so")
CFLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
          "-Wall", "-Wextra"]

_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle into oracle/libdmsgm_oracle.so (gcc, no FMA contraction)."""
    newest = max(os.path.getmtime(f) for f in (_SRC, _SRC2, _SRC3, _SRC4, _HDR, _HDR2))
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < newest:
        tmp = LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, _SRC4, _SRC2, _SRC3, "-lm"])
        os.replace(tmp, LIB_PATH)
    return LIB_PATH


class _Params(ctypes.Structure):
    _fields_ = [("theta_s", ctypes.c_float), ("theta_d", ctypes.c_float),
                ("var_init", ctypes.c_float), ("age_cap", ctypes.c_float),
                ("var_floor_match", ctypes.c_float), ("var_floor_classify", ctypes.c_float),
                ("decay_lambda", ctypes.c_float), ("decay_var_thresh", ctypes.c_float),
                ("num_streams", ctypes.c_int), ("update_rule", ctypes.c_int),
                ("classify_rule", ctypes.c_int), ("form", ctypes.c_int)]

FORM_KERNEL_ORDER = 0   # dmsgm_oracle.c: the canonical fp32 order the CUDA path reproduces bitwise
FORM_PLAIN = 1          # dmsgm_plain.c: SURVEY §8(c)'s literal definition (fp64 projection, / sum W, libm exp)


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            P = ctypes.c_void_p
            i32, sz = ctypes.c_int, ctypes.c_size_t
            lib.dmsgm_oracle_create.argtypes = [i32, i32, i32, ctypes.POINTER(_Params),
                                                ctypes.POINTER(P)]
            lib.dmsgm_oracle_destroy.argtypes = [P]
            lib.dmsgm_oracle_destroy.restype = None
            lib.dmsgm_oracle_step.argtypes = [P, P, sz, P, P, sz]
            lib.dmsgm_oracle_step_stream.argtypes = [P, i32, P, sz, P, P, sz]
            lib.dmsgm_oracle_commit.argtypes = [P]
            lib.dmsgm_oracle_reset.argtypes = [P, i32]
            lib.dmsgm_oracle_get_state.argtypes = [P, i32, P]
            lib.dmsgm_oracle_set_state.argtypes = [P, i32, P]
            lib.dmsgm_oracle_is_initialised.argtypes = [P, i32]
            lib.dmsgm_oracle_mix_weights.argtypes = [i32, i32, i32, P, i32, i32, P, P, P, P]
            lib.dmsgm_oracle_decay_factor.argtypes = [ctypes.c_float, ctypes.c_float]
            lib.dmsgm_oracle_decay_factor.restype = ctypes.c_float
            lib.dmsgm_oracle_set_tilde_probe.argtypes = [P, P]
            lib.dmsgm_oracle_gauss_taps.argtypes = [i32, ctypes.c_float, P]
            lib.dmsgm_oracle_prefilter.argtypes = [i32, i32, P, sz, P, sz, i32, ctypes.c_float, i32]
            lib.dmsgm_oracle_warp_frame.argtypes = [i32, i32, P, sz, P, P, sz]
            _lib = lib
    return _lib


@dataclass
class OracleParams:
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
    form: int = FORM_KERNEL_ORDER

    def _c(self) -> _Params:
        return _Params(self.theta_s, self.theta_d, self.var_init, self.age_cap,
                       self.var_floor_match, self.var_floor_classify, self.decay_lambda,
                       self.decay_var_thresh, self.num_streams, self.update_rule,
                       self.classify_rule, self.form)


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


class Oracle:
    """One oracle context: S streams of WxH frames with NxN blocks (host memory)."""

    def __init__(self, width: int, height: int, block: int, params: OracleParams):
        self.lib = _load()
        self.W, self.H, self.N = width, height, block
        self.Wb, self.Hb = width // block, height // block
        self.params = params
        self.S = params.num_streams
        h = ctypes.c_void_p()
        cp = params._c()
        rc = self.lib.dmsgm_oracle_create(width, height, block, ctypes.byref(cp), ctypes.byref(h))
        if rc != 0:
            raise ValueError(f"dmsgm_oracle_create failed ({rc})")
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            self.lib.dmsgm_oracle_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def step(self, frames: np.ndarray, homographies: np.ndarray) -> np.ndarray:
        """frames u8 [S][H][W] (C-contiguous), homographies f64 [S][9] -> masks u8 [S][H][W]."""
        frames = np.ascontiguousarray(frames, np.uint8)
        Hs = np.ascontiguousarray(homographies, np.float64)
        assert frames.shape == (self.S, self.H, self.W), frames.shape
        assert Hs.shape == (self.S, 9), Hs.shape
        masks = np.empty_like(frames)
        rc = self.lib.dmsgm_oracle_step(self._h, _ptr(frames), self.W, _ptr(Hs), _ptr(masks), self.W)
        if rc != 0:
            raise RuntimeError(f"dmsgm_oracle_step failed ({rc})")
        return masks

    def step_stream(self, s: int, frame: np.ndarray, homography: np.ndarray, mask: np.ndarray):
        """Step one stream (thread-safe across distinct s; ctypes drops the GIL)."""
        rc = self.lib.dmsgm_oracle_step_stream(self._h, s, _ptr(frame), self.W, _ptr(homography),
                                               _ptr(mask), self.W)
        if rc != 0:
            raise RuntimeError(f"dmsgm_oracle_step_stream failed ({rc})")

    def commit(self):
        self.lib.dmsgm_oracle_commit(self._h)

    def reset(self, stream: int = -1):
        if self.lib.dmsgm_oracle_reset(self._h, stream) != 0:
            raise ValueError("bad stream")

    def get_state(self, stream: int) -> np.ndarray:
        out = np.empty((6, self.Hb, self.Wb), np.float32)
        if self.lib.dmsgm_oracle_get_state(self._h, stream, _ptr(out)) != 0:
            raise ValueError("bad stream")
        return out

    def set_state(self, stream: int, state: np.ndarray):
        st = np.ascontiguousarray(state, np.float32)
        assert st.shape == (6, self.Hb, self.Wb)
        if self.lib.dmsgm_oracle_set_state(self._h, stream, _ptr(st)) != 0:
            raise ValueError("bad stream")

    def set_tilde_probe(self, on: bool = True):
        """While on, every step records per block the tilde models after S1-S3, M and a
        live flag into self.tilde [S][8][Hb][Wb] (test probe)."""
        if on:
            self.tilde = np.zeros((self.S, 8, self.Hb, self.Wb), np.float32)
            self.lib.dmsgm_oracle_set_tilde_probe(self._h, _ptr(self.tilde))
        else:
            self.lib.dmsgm_oracle_set_tilde_probe(self._h, None)

    def is_initialised(self, stream: int) -> bool:
        return bool(self.lib.dmsgm_oracle_is_initialised(self._h, stream))


def decay_factor(lam: float, d: float) -> float:
    """exp(-lam * d) as the kernel-order form evaluates it (reading R18), lam and d fp32."""
    return float(_load().dmsgm_oracle_decay_factor(lam, d))


def gauss_taps(size: int, sigma: float) -> np.ndarray:
    """The normalised fp32 Gaussian taps of reading R30."""
    t = np.zeros(size, np.float32)
    if _load().dmsgm_oracle_gauss_taps(size, sigma, _ptr(t)) != 0:
        raise ValueError("bad taps arguments")
    return t


def prefilter(frame: np.ndarray, gauss_size: int = 5, gauss_sigma: float = 1.0, median_radius: int = 1) -> np.ndarray:
    """§2.1 preprocessing of one u8 frame [H][W] (readings R30-R34): separable Gaussian, then median."""
    f = np.ascontiguousarray(frame, np.uint8)
    H, W = f.shape
    out = np.empty_like(f)
    if _load().dmsgm_oracle_prefilter(W, H, _ptr(f), W, _ptr(out), W, gauss_size, gauss_sigma, median_radius) != 0:
        raise ValueError("bad prefilter arguments")
    return out


def prefilter_frames(frames: np.ndarray, gauss_size: int = 5, gauss_sigma: float = 1.0,
                     median_radius: int = 1) -> np.ndarray:
    """prefilter() over [..., H, W]."""
    out = np.empty_like(frames)
    flat_in = frames.reshape(-1, *frames.shape[-2:])
    flat_out = out.reshape(-1, *frames.shape[-2:])
    for i in range(flat_in.shape[0]):
        flat_out[i] = prefilter(flat_in[i], gauss_size, gauss_sigma, median_radius)
    return out


def warp_frame(frame: np.ndarray, h) -> np.ndarray:
    """App. F frame-warp motion compensation of one u8 frame [H][W] (readings R35-R37)."""
    f = np.ascontiguousarray(frame, np.uint8)
    hh = np.ascontiguousarray(np.asarray(h, np.float64).reshape(9))
    Hh, W = f.shape
    out = np.empty_like(f)
    if _load().dmsgm_oracle_warp_frame(W, Hh, _ptr(f), W, _ptr(hh), _ptr(out), W) != 0:
        raise ValueError("bad warp arguments")
    return out


def warp_frames(frames: np.ndarray, homographies: np.ndarray) -> np.ndarray:
    """warp_frame over [..., H, W] frames with [..., 9] homographies."""
    out = np.empty_like(frames)
    fi = frames.reshape(-1, *frames.shape[-2:])
    hi = homographies.reshape(-1, 9)
    fo = out.reshape(-1, *frames.shape[-2:])
    for i in range(fi.shape[0]):
        fo[i] = warp_frame(fi[i], hi[i])
    return out


def mix_weights(width: int, height: int, block: int, h, bi: int, bj: int, with_clipped: bool = False):
    """Step S1 for one block: (exposed, src [(x,y)]*4, raw weights f32[4], sumW[, clipped])."""
    lib = _load()
    hh = np.ascontiguousarray(np.asarray(h, np.float64).reshape(9))
    sx = np.zeros(4, np.int32)
    sy = np.zeros(4, np.int32)
    w = np.zeros(4, np.float32)
    sw = np.zeros(1, np.float32)
    rc = lib.dmsgm_oracle_mix_weights(width, height, block, _ptr(hh), bi, bj, _ptr(sx), _ptr(sy),
                                      _ptr(w), _ptr(sw))
    if rc < 0:
        raise ValueError("bad arguments")
    out = (rc == 1, list(zip(sx.tolist(), sy.tolist())), w, float(sw[0]))
    return out + (rc == 2,) if with_clipped else out


def run_sequence(frames: np.ndarray, homographies: np.ndarray, block: int,
                 params: OracleParams, states_at=()):
    """Run the oracle over frames [T][S][H][W]; returns (masks [T][S][H][W], final states [S][6][Hb][Wb],
    {t: states} for t in states_at)."""
    T, S, H, W = frames.shape
    p = OracleParams(**{**params.__dict__, "num_streams": S})
    o = Oracle(W, H, block, p)
    masks = np.empty_like(frames)
    snaps = {}
    for t in range(T):
        masks[t] = o.step(frames[t], homographies[t])
        if t in states_at:
            snaps[t] = np.stack([o.get_state(s) for s in range(S)])
    final = np.stack([o.get_state(s) for s in range(S)])
    o.close()
    return masks, final, snaps
