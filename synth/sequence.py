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
def _hash_u01(ix: np.ndarray, iy: np.ndarray, seed: int) -> np.ndarray:
    """Counter-based hash of integer lattice coords -> [-1, 1)."""
    m = np.uint64(0xFFFFFFFF)
    h = (ix.astype(np.int64).astype(np.uint64) * np.uint64(0x9E3779B1)
         + iy.astype(np.int64).astype(np.uint64) * np.uint64(0x85EBCA77)
         + np.uint64(seed) * np.uint64(0xC2B2AE3D)) & m
    h ^= h >> np.uint64(15)
    h = (h * np.uint64(0x2C1B3C6D)) & m
    h ^= h >> np.uint64(12)
    h = (h * np.uint64(0x297A2D39)) & m
    h ^= h >> np.uint64(15)
    return (h.astype(np.float64) / 4294967296.0 * 2.0 - 1.0).astype(np.float32)


def _texture(wx: np.ndarray, wy: np.ndarray, sp: _StreamParams) -> np.ndarray:
    acc = np.zeros(wx.shape, np.float32)
    for k in range(6):
        c, s = math.cos(sp.tex_dirs[k]), math.sin(sp.tex_dirs[k])
        f = np.float32(2 * math.pi / sp.tex_periods[k])
        acc += np.sin((wx * np.float32(c) + wy * np.float32(s)) * f + np.float32(sp.tex_phases[k]))
    gx, gy = wx / np.float32(8.0), wy / np.float32(8.0)
    ix, iy = np.floor(gx), np.floor(gy)
    fx, fy = gx - ix, gy - iy
    ix, iy = ix.astype(np.int64), iy.astype(np.int64)
    n00 = _hash_u01(ix, iy, sp.lattice_seed)
    n10 = _hash_u01(ix + 1, iy, sp.lattice_seed)
    n01 = _hash_u01(ix, iy + 1, sp.lattice_seed)
    n11 = _hash_u01(ix + 1, iy + 1, sp.lattice_seed)
    noise = (n00 * (1 - fx) + n10 * fx) * (1 - fy) + (n01 * (1 - fx) + n11 * fx) * fy
    t = np.clip(np.float32(0.25) * acc + np.float32(0.45) * noise, -1.0, 1.0)
    return np.float32(125.0) + np.float32(95.0) * t


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
                 want_gt: bool = False):
    """Render frame t of a stream: returns (u8 [H][W], gt u8 [H][W] or None)."""
    P = camera_pose(cfg, sp, t)
    xs = np.arange(cfg.W, dtype=np.float64) + 0.5
    ys = np.arange(cfg.H, dtype=np.float64) + 0.5
    X, Y = np.meshgrid(xs, ys)
    w = P[2, 0] * X + P[2, 1] * Y + P[2, 2]
    wx = ((P[0, 0] * X + P[0, 1] * Y + P[0, 2]) / w).astype(np.float32)
    wy = ((P[1, 0] * X + P[1, 1] * Y + P[1, 2]) / w).astype(np.float32)
    img = _texture(wx, wy, sp)
    gt = np.zeros((cfg.H, cfg.W), np.uint8) if want_gt else None
    for o in sp.objects:
        c = _object_pos(cfg, o, t)
        if o["kind"] == "disc":
            inside = (X - c[0]) ** 2 + (Y - c[1]) ** 2 <= (o["w"] / 2) ** 2
        else:
            inside = (np.abs(X - c[0]) <= o["w"] / 2) & (np.abs(Y - c[1]) <= o["h"] / 2)
        img[inside] = o["I"]
        if want_gt:
            gt[inside] = 255
    if cfg.noise > 0:
        nrng = np.random.default_rng((sp.noise_seed, t))
        img = img + nrng.normal(0.0, cfg.noise, img.shape).astype(np.float32)
    out = np.clip(np.rint(img), 0, 255).astype(np.uint8)
    return out, gt


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
    for j, s in enumerate(streams):
        sp = _stream_params(cfg, s)
        Hs[:, j] = homographies_for_stream(cfg, s, T, sp)
        for t in range(T):
            f, g = render_frame(cfg, sp, t, s, with_gt)
            frames[t, j] = f
            if with_gt:
                gts[t, j] = g
    return Sequence(cfg, frames, Hs, gts)
