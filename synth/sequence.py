"""Seeded synthetic video sequences with known camera homographies.

Recipe (SURVEY.md §8(d) "Configs restated as synthetic inputs"):

* background: a procedural world texture -- 6 random-direction sinusoids with
  periods 6..64 px plus an 8-px value-noise lattice (counter-hash, bilinear) --
  mapped to [30, 220] and sampled at pixel centres (x+1/2, y+1/2) through the
  camera pose P_t (frame-t pixel coords -> world coords);
* foreground: constant-intensity squares / rectangles / discs (contrast >= 60
  against the mid-grey background) moving with constant image velocity and
  reflecting at the borders (or on closed orbits in ``ring`` mode);
* additive N(0, noise^2) sensor noise, rounded and clamped to [0, 255];
* homographies H_t = P_{t-1}^{-1} P_t (maps frame-t coords to frame-(t-1)
  coords, reading R3), normalised to h8 = 1.  H_0 is the identity (the first
  frame initialises the model and ignores H), except in ``ring`` mode where the
  sequence is periodic and H_0 = P_{R-1}^{-1} P_0.

RNG: numpy ``default_rng(seed + stream)``.  Nothing here computes any part of
the DMSGM method.
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass, field, replace
from typing import Optional

import numpy as np

_DEG = math.pi / 180.0


@dataclass(frozen=True)
class SeqConfig:
    name: str
    W: int
    H: int
    N: int            # model block size (not used by the generator; carried for callers)
    S: int            # number of independent streams
    T: int            # number of frames
    seed: int
    noise: float      # sensor noise sigma (grey levels)
    camera: str       # "identity" | "pan_rot" | "pan_zoom_sin" | "random" | "ring"
    pan: tuple = (0.0, 0.0)          # px/frame (pan_rot) or max |v| per axis (random)
    rot_deg: float = 0.0             # deg/frame (pan_rot) or max |omega| (random)
    zoom: float = 0.0                # max |z-1| per frame (random) or sin amplitude (pan_zoom_sin)
    n_objects: tuple = (1, 1)        # inclusive range of objects per stream
    objects: Optional[tuple] = None  # explicit object list (overrides random objects)
    period: int = 0                  # ring period (frames) for camera == "ring"


# The five BASELINE.json configs.  C4/C5 "ring" variants
# are the bench workloads: same per-frame motion statistics, periodic so a ring of
# R distinct frames per stream can be cycled without a seam.
CONFIGS = {
    "C1": SeqConfig("C1", 64, 48, 4, 1, 10, 11, 0.0, "identity",
                    objects=(("square", 8, 8, 230, 8.0, 8.0, 4.0, 2.0),)),
    "C2": SeqConfig("C2", 320, 240, 4, 1, 300, 21, 2.0, "pan_rot", pan=(0.7, -0.3),
                    rot_deg=0.05,
                    objects=(("rect", 24, 16, 220, 60.0, 50.0, 1.5, 0.8),
                             ("disc", 10, 10, 25, 200.0, 150.0, -1.1, 0.9))),
    "C3": SeqConfig("C3", 640, 480, 4, 1, 1000, 31, 2.0, "pan_zoom_sin", pan=(1.0, 0.6),
                    zoom=0.05, n_objects=(5, 5)),
    "C4": SeqConfig("C4", 1920, 1080, 4, 32, 300, 4000, 2.0, "random", pan=(2.0, 2.0),
                    rot_deg=0.05, zoom=0.0005, n_objects=(4, 8)),
    "C5": SeqConfig("C5", 3840, 2160, 8, 64, 100, 5000, 2.0, "random", pan=(4.0, 4.0),
                    rot_deg=0.05, zoom=0.0005, n_objects=(4, 8)),
    "C4ring": SeqConfig("C4ring", 1920, 1080, 4, 32, 8, 4000, 2.0, "ring", pan=(2.0, 2.0),
                        rot_deg=0.05, zoom=0.0005, n_objects=(4, 8), period=8),
    "C5ring": SeqConfig("C5ring", 3840, 2160, 8, 64, 8, 5000, 2.0, "ring", pan=(4.0, 4.0),
                        rot_deg=0.05, zoom=0.0005, n_objects=(4, 8), period=8),
    # C4p: the paper's own per-pixel DSGM (block = 1) at 1080p, 4 streams
    "C4pring": SeqConfig("C4pring", 1920, 1080, 1, 4, 8, 4100, 2.0, "ring", pan=(2.0, 2.0),
                         rot_deg=0.05, zoom=0.0005, n_objects=(4, 8), period=8),
    # C5b: ONE 4K stream split into row bands over the GPUs; motion
    # small enough (pan <= 2 px, rotation <= 0.02 deg per frame) for a one-block-row halo
    "C5b": SeqConfig("C5b", 3840, 2160, 8, 1, 100, 5100, 2.0, "random", pan=(2.0, 2.0),
                     rot_deg=0.02, zoom=0.0005, n_objects=(6, 6)),
    "C5bring": SeqConfig("C5bring", 3840, 2160, 8, 1, 8, 5100, 2.0, "ring", pan=(2.0, 2.0),
                         rot_deg=0.02, zoom=0.0005, n_objects=(6, 6), period=8),
}


def config(name: str, **overrides) -> SeqConfig:
    """Return a named config, optionally with fields replaced (e.g. T=3, S=2)."""
    return replace(CONFIGS[name], **overrides)


@dataclass
class Sequence:
    cfg: SeqConfig
    frames: np.ndarray        # u8  [T][S][H][W]
    homographies: np.ndarray  # f64 [T][S][9]
    gt: Optional[np.ndarray]  # u8  [T][S][H][W] in {0,255} or None


def stream_rng(cfg: SeqConfig, s: int) -> np.random.Generator:
    return np.random.default_rng(cfg.seed + s)


# ---------------------------------------------------------------------------
# per-stream random parameters (drawn in a fixed order from stream_rng)
# ---------------------------------------------------------------------------
@dataclass
class _StreamParams:
    tex_dirs: np.ndarray
    tex_periods: np.ndarray
    tex_phases: np.ndarray
    lattice_seed: int
    cam: dict
    objects: list = field(default_factory=list)
    noise_seed: int = 0


def _stream_params(cfg: SeqConfig, s: int) -> _StreamParams:
    rng = stream_rng(cfg, s)
    dirs = rng.uniform(0.0, math.pi, 6)
    periods = rng.uniform(6.0, 64.0, 6)
    phases = rng.uniform(0.0, 2 * math.pi, 6)
    lattice_seed = int(rng.integers(0, 2**31 - 1))
    cam = {}
    if cfg.camera in ("random", "ring"):
        cam["v"] = rng.uniform(-1.0, 1.0, 2) * np.asarray(cfg.pan, dtype=np.float64)
        cam["omega"] = rng.uniform(-1.0, 1.0) * cfg.rot_deg * _DEG
        cam["z"] = 1.0 + rng.uniform(-1.0, 1.0) * cfg.zoom
        cam["phase"] = rng.uniform(0.0, 2 * math.pi, 3)
    objs = []
    if cfg.objects is not None:
        for (kind, w, h, inten, x, y, vx, vy) in cfg.objects:
            objs.append(dict(kind=kind, w=float(w), h=float(h), I=int(inten),
                             p=np.array([x, y]), v=np.array([vx, vy]),
                             orbit=None))
    else:
        lo, hi = cfg.n_objects
        n = int(rng.integers(lo, hi + 1))
        for _ in range(n):
            kind = ("square", "rect", "disc")[int(rng.integers(0, 3))]
            size = max(8.0, 0.03 * min(cfg.W, cfg.H)) * rng.uniform(1.0, 2.5)
            w = size
            h = size * (rng.uniform(0.5, 1.0) if kind == "rect" else 1.0)
            dark = bool(rng.integers(0, 2))
            inten = int(rng.integers(5, 40)) if dark else int(rng.integers(215, 251))
            p = np.array([rng.uniform(w, cfg.W - w), rng.uniform(h, cfg.H - h)])
            speed = rng.uniform(0.5, 3.0)
            ang = rng.uniform(0, 2 * math.pi)
            v = speed * np.array([math.cos(ang), math.sin(ang)])
            orbit = None
            if cfg.camera == "ring":
                orbit = dict(r=speed * cfg.period / (2 * math.pi), ph=ang)
            objs.append(dict(kind=kind, w=w, h=h, I=inten, p=p, v=v, orbit=orbit))
    noise_seed = int(rng.integers(0, 2**31 - 1))
    return _StreamParams(dirs, periods, phases, lattice_seed, cam, objs, noise_seed)


# ---------------------------------------------------------------------------
# camera
# ---------------------------------------------------------------------------
def _tr(x, y):
    return np.array([[1.0, 0.0, x], [0.0, 1.0, y], [0.0, 0.0, 1.0]])


def _rot(th):
    c, s = math.cos(th), math.sin(th)
    return np.array([[c, -s, 0.0], [s, c, 0.0], [0.0, 0.0, 1.0]])


def _scale(z):
    return np.array([[z, 0.0, 0.0], [0.0, z, 0.0], [0.0, 0.0, 1.0]])


def camera_pose(cfg: SeqConfig, sp: _StreamParams, t: int) -> np.ndarray:
    """P_t: frame-t pixel coordinates -> world coordinates (3x3, float64)."""
    cx, cy = cfg.W / 2.0, cfg.H / 2.0
    if cfg.camera == "identity":
        return np.eye(3)
    if cfg.camera == "pan_rot":
        d = np.array(cfg.pan) * t
        th = cfg.rot_deg * _DEG * t
        z = 1.0
    elif cfg.camera == "pan_zoom_sin":
        # velocity amplitude cfg.pan px/frame, period 200 -> displacement amplitude pan*200/2pi
        amp = np.array(cfg.pan) * 200.0 / (2 * math.pi)
        d = amp * np.array([math.sin(2 * math.pi * t / 200.0), 1.0 - math.cos(2 * math.pi * t / 200.0)])
        th = 0.0
        z = 1.0 + cfg.zoom * math.sin(2 * math.pi * t / 500.0)
    elif cfg.camera == "random":
        d = sp.cam["v"] * t
        th = sp.cam["omega"] * t
        z = sp.cam["z"] ** t
    elif cfg.camera == "ring":
        R = cfg.period
        ph = sp.cam["phase"]
        k = 2 * math.pi / R
        # peak per-frame speed ~ |v|, |omega|, |z-1| of the "random" recipe
        d = sp.cam["v"] / k * np.array([math.sin(k * t + ph[0]), math.sin(k * t + ph[0] + 1.0)])
        th = sp.cam["omega"] / k * math.sin(k * t + ph[1])
        z = 1.0 + (sp.cam["z"] - 1.0) / k * math.sin(k * t + ph[2])
    else:
        raise ValueError(cfg.camera)
    return _tr(cx + d[0], cy + d[1]) @ _rot(th) @ _scale(z) @ _tr(-cx, -cy)


def homographies_for_stream(cfg: SeqConfig, s: int, T: Optional[int] = None,
                            sp: Optional[_StreamParams] = None) -> np.ndarray:
    """[T][9] float64, H_t = P_{t-1}^{-1} P_t normalised to h8 = 1 (reading R3)."""
    T = cfg.T if T is None else T
    sp = _stream_params(cfg, s) if sp is None else sp
    out = np.zeros((T, 9))
    for t in range(T):
        if t == 0 and cfg.camera != "ring":
            Hm = np.eye(3)
        else:
            tp = (t - 1) % cfg.period if cfg.camera == "ring" else t - 1
            Hm = np.linalg.solve(camera_pose(cfg, sp, tp), camera_pose(cfg, sp, t))
            Hm = Hm / Hm[2, 2]
        out[t] = Hm.reshape(9)
    return out


# ---------------------------------------------------------------------------
# texture + objects
# ---------------------------------------------------------------------------
class _NP:
    """numpy backend (reference inputs for the parity tests)."""
    name = "numpy"

    def __init__(self):
        self.f32 = np.float32

    def grid(self, W, H):
        xs = np.arange(W, dtype=np.float64) + 0.5
        ys = np.arange(H, dtype=np.float64) + 0.5
        return np.meshgrid(xs, ys)

    def to_f32(self, a):
        return a.astype(np.float32)

    def i64(self, a):
        return a.astype(np.int64)

    sin = staticmethod(np.sin)
    floor = staticmethod(np.floor)
    abs = staticmethod(np.abs)

    def clip(self, a, lo, hi):
        return np.clip(a, lo, hi)

    def zeros_u8(self, H, W):
        return np.zeros((H, W), np.uint8)

    def noise(self, seed_tuple, shape, sigma):
        return np.random.default_rng(seed_tuple).normal(0.0, sigma, shape).astype(np.float32)

    def to_u8(self, img):
        return np.clip(np.rint(img), 0, 255).astype(np.uint8)


class _Torch:
    """torch backend (fast bench inputs, e.g. on cuda); same recipe, different rounding/noise."""
    name = "torch"

    def __init__(self, device):
        import torch
        self.t = torch
        self.device = torch.device(device)
        self.f32 = torch.float32

    def grid(self, W, H):
        t = self.t
        xs = t.arange(W, dtype=t.float64, device=self.device) + 0.5
        ys = t.arange(H, dtype=t.float64, device=self.device) + 0.5
        Y, X = t.meshgrid(ys, xs, indexing="ij")
        return X, Y

    def to_f32(self, a):
        return a.to(self.t.float32)

    def i64(self, a):
        return a.to(self.t.int64)

    def sin(self, a):
        return self.t.sin(a)

    def floor(self, a):
        return self.t.floor(a)

    def abs(self, a):
        return self.t.abs(a)

    def clip(self, a, lo, hi):
        return self.t.clamp(a, lo, hi)

    def zeros_u8(self, H, W):
        return self.t.zeros((H, W), dtype=self.t.uint8, device=self.device)

    def noise(self, seed_tuple, shape, sigma):
        g = self.t.Generator(device=self.device)
        g.manual_seed((int(seed_tuple[0]) * 1000003 + int(seed_tuple[1])) % (2**63 - 1))
        return self.t.randn(shape, generator=g, device=self.device, dtype=self.t.float32) * sigma

    def to_u8(self, img):
        return self.t.clamp(self.t.round(img), 0, 255).to(self.t.uint8)


_NUMPY = _NP()


def _hash_u01(bk, ix, iy, seed: int):
    """Counter-based hash of integer lattice coords -> [-1, 1) (identical low bits on both backends)."""
    m = 0xFFFFFFFF
    h = (ix * 0x9E3779B1 + iy * 0x85EBCA77 + (seed * 0xC2B2AE3D & m)) & m
    h = h ^ (h >> 15)
    h = (h * 0x2C1B3C6D) & m
    h = h ^ (h >> 12)
    h = (h * 0x297A2D39) & m
    h = h ^ (h >> 15)
    return bk.to_f32(h) * (2.0 / 4294967296.0) - 1.0


def _texture(bk, wx, wy, sp: _StreamParams):
    acc = None
    for k in range(6):
        c, s = math.cos(sp.tex_dirs[k]), math.sin(sp.tex_dirs[k])
        f = 2 * math.pi / sp.tex_periods[k]
        term = bk.sin((wx * c + wy * s) * f + sp.tex_phases[k])
        acc = term if acc is None else acc + term
    gx, gy = wx * 0.125, wy * 0.125
    fx0, fy0 = bk.floor(gx), bk.floor(gy)
    fx, fy = gx - fx0, gy - fy0
    ix, iy = bk.i64(fx0) & 0xFFFFFFFF, bk.i64(fy0) & 0xFFFFFFFF
    n00 = _hash_u01(bk, ix, iy, sp.lattice_seed)
    n10 = _hash_u01(bk, (ix + 1) & 0xFFFFFFFF, iy, sp.lattice_seed)
    n01 = _hash_u01(bk, ix, (iy + 1) & 0xFFFFFFFF, sp.lattice_seed)
    n11 = _hash_u01(bk, (ix + 1) & 0xFFFFFFFF, (iy + 1) & 0xFFFFFFFF, sp.lattice_seed)
    noise = (n00 * (1 - fx) + n10 * fx) * (1 - fy) + (n01 * (1 - fx) + n11 * fx) * fy
    t = bk.clip(acc * 0.25 + noise * 0.45, -1.0, 1.0)
    return t * 95.0 + 125.0


def _reflect(x: float, lo: float, hi: float) -> float:
    span = hi - lo
    if span <= 0:
        return lo
    y = (x - lo) % (2 * span)
    return lo + (y if y <= span else 2 * span - y)


def _object_pos(cfg: SeqConfig, o: dict, t: int) -> np.ndarray:
    if o["orbit"] is not None:
        k = 2 * math.pi / cfg.period
        r, ph = o["orbit"]["r"], o["orbit"]["ph"]
        c = o["p"]
        return np.array([c[0] + r * math.cos(k * t + ph), c[1] + r * math.sin(k * t + ph)])
    p = o["p"] + o["v"] * t
    return np.array([_reflect(p[0], o["w"] / 2, cfg.W - o["w"] / 2),
                     _reflect(p[1], o["h"] / 2, cfg.H - o["h"] / 2)])


def render_frame(cfg: SeqConfig, sp: _StreamParams, t: int, s: int = 0,
                 want_gt: bool = False, backend=None):
    """Render frame t of a stream: returns (u8 [H][W], gt u8 [H][W] or None).

    backend: None/numpy (default, the parity-test reference) or a torch device string.
    """
    bk = _NUMPY if backend is None or backend == "numpy" else _Torch(backend)
    P = camera_pose(cfg, sp, t)
    X, Y = bk.grid(cfg.W, cfg.H)
    w = X * P[2, 0] + Y * P[2, 1] + P[2, 2]
    wx = bk.to_f32((X * P[0, 0] + Y * P[0, 1] + P[0, 2]) / w)
    wy = bk.to_f32((X * P[1, 0] + Y * P[1, 1] + P[1, 2]) / w)
    img = _texture(bk, wx, wy, sp)
    gt = bk.zeros_u8(cfg.H, cfg.W) if want_gt else None
    for o in sp.objects:
        c = _object_pos(cfg, o, t)
        if o["kind"] == "disc":
            inside = (X - c[0]) ** 2 + (Y - c[1]) ** 2 <= (o["w"] / 2) ** 2
        else:
            inside = (bk.abs(X - c[0]) <= o["w"] / 2) & (bk.abs(Y - c[1]) <= o["h"] / 2)
        img[inside] = float(o["I"])
        if want_gt:
            gt[inside] = 255
    if cfg.noise > 0:
        img = img + bk.noise((sp.noise_seed, t), tuple(img.shape), cfg.noise)
    return bk.to_u8(img), gt


def generate_device(cfg, T: Optional[int] = None, streams=None, device: str = "cuda"):
    """Fast torch variant of generate() for the bench: (frames u8 [T][S'][H][W] on `device`,
    homographies f64 [T][S'][9] numpy).  Same recipe; pixel values differ from the numpy
    backend in rounding and noise draws (bench inputs are not parity references)."""
    import torch
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    T = cfg.T if T is None else T
    streams = list(range(cfg.S)) if streams is None else list(streams)
    frames = torch.empty((T, len(streams), cfg.H, cfg.W), dtype=torch.uint8, device=device)
    Hs = np.empty((T, len(streams), 9))
    for j, s in enumerate(streams):
        sp = _stream_params(cfg, s)
        Hs[:, j] = homographies_for_stream(cfg, s, T, sp)
        for t in range(T):
            frames[t, j] = render_frame(cfg, sp, t, s, False, backend=device)[0]
    return frames, Hs


def generate(cfg, T: Optional[int] = None, streams=None, with_gt: bool = False) -> Sequence:
    """Generate frames [T][S'][H][W], homographies [T][S'][9] (and GT masks).

    ``streams`` selects a subset of stream indices (default: all cfg.S); each
    stream depends only on (cfg.seed + s), so subsets are consistent.
    """
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    T = cfg.T if T is None else T
    streams = list(range(cfg.S)) if streams is None else list(streams)
    frames = np.empty((T, len(streams), cfg.H, cfg.W), np.uint8)
    Hs = np.empty((T, len(streams), 9))
    gts = np.empty((T, len(streams), cfg.H, cfg.W), np.uint8) if with_gt else None
    jobs = []
    for j, s in enumerate(streams):
        sp = _stream_params(cfg, s)
        Hs[:, j] = homographies_for_stream(cfg, s, T, sp)
        jobs += [(j, s, sp, t) for t in range(T)]

    def render(job):
        j, s, sp, t = job
        f, g = render_frame(cfg, sp, t, s, with_gt)
        frames[t, j] = f
        if with_gt:
            gts[t, j] = g

    # frames are independent (per-frame noise seeds), so they render in parallel threads
    # (numpy releases the GIL); the bytes do not depend on the thread count
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=max(1, min(16, os.cpu_count() or 1))) as ex:
        list(ex.map(render, jobs))
    return Sequence(cfg, frames, Hs, gts)
