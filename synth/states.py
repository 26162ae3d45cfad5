"""Seeded random model states and homographies (inputs only, no DMSGM arithmetic).

State layout used by both sides' get/set_state: float32 [6][Hb][Wb] per stream,
planes in the order (mu_A, var_A, age_A, mu_C, var_C, age_C) -- DESIGN.md §3.
"""
from __future__ import annotations

import math

import numpy as np


def blocks_of(W: int, H: int, N: int):
    """(Wb, Hb): block-grid shape for an HxW frame with NxN blocks (reading R1)."""
    return W // N, H // N


def random_state(rng: np.random.Generator, Hb: int, Wb: int, age_cap: float = 30.0,
                 integer_ages: bool = False, var_max: float = 4000.0,
                 special: bool = True) -> np.ndarray:
    """A valid random state [6][Hb][Wb] (mu in [0,255], var >= 0, 0 < age <= cap).

    With ``special`` some entries are set to awkward values: integer and
    half-integer means, tiny variances, ages at the cap, equal A/C ages.
    """
    st = np.empty((6, Hb, Wb), np.float32)
    for m in (0, 3):
        st[m] = rng.uniform(0.0, 255.0, (Hb, Wb))
        st[m + 1] = np.exp(rng.uniform(math.log(0.01), math.log(var_max), (Hb, Wb)))
        if integer_ages:
            st[m + 2] = rng.integers(1, int(age_cap) + 1, (Hb, Wb))
        else:
            st[m + 2] = rng.uniform(1.0, age_cap, (Hb, Wb))
    if special:
        sel = rng.random((Hb, Wb))
        st[0][sel < 0.1] = np.rint(st[0][sel < 0.1])
        st[0][(sel >= 0.1) & (sel < 0.2)] = np.floor(st[0][(sel >= 0.1) & (sel < 0.2)]) + 0.5
        st[1][(sel >= 0.2) & (sel < 0.3)] = rng.uniform(0.0, 0.3, int(((sel >= 0.2) & (sel < 0.3)).sum()))
        st[2][(sel >= 0.3) & (sel < 0.4)] = age_cap
        st[5][(sel >= 0.4) & (sel < 0.5)] = st[2][(sel >= 0.4) & (sel < 0.5)]
    return st


def random_homography(rng: np.random.Generator, W: int, H: int, shift: float = 3.0,
                      rot_deg: float = 0.5, zoom: float = 0.01, persp: float = 1e-5) -> np.ndarray:
    """A random near-identity homography about the image centre, h8 = 1, as [9]."""
    cx, cy = W / 2.0, H / 2.0
    th = rng.uniform(-rot_deg, rot_deg) * math.pi / 180.0
    z = 1.0 + rng.uniform(-zoom, zoom)
    c, s = math.cos(th), math.sin(th)
    A = np.array([[z * c, -z * s, 0.0], [z * s, z * c, 0.0], [0.0, 0.0, 1.0]])
    T1 = np.array([[1.0, 0.0, -cx], [0.0, 1.0, -cy], [0.0, 0.0, 1.0]])
    T2 = np.array([[1.0, 0.0, cx + rng.uniform(-shift, shift)],
                   [0.0, 1.0, cy + rng.uniform(-shift, shift)], [0.0, 0.0, 1.0]])
    P = np.eye(3)
    P[2, 0] = rng.uniform(-persp, persp)
    P[2, 1] = rng.uniform(-persp, persp)
    Hm = T2 @ A @ T1
    Hm = P @ Hm
    return (Hm / Hm[2, 2]).reshape(9)
