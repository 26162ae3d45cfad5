"""Pins for the motion-estimation oracle (oracle/klt_oracle.py, SURVEY §8(f) NEXT-4;
PAPER.md App. F, SPEC S:278-313 fixtures).

Each test checks the oracle against something other than itself: library routines
(scipy.ndimage, numpy.linalg), closed forms, constructed ground truth (shifted images,
forward-generated correspondences), published values, and the defining invariants of the
greedy corner selection.
"""
import math

import numpy as np
import pytest
from scipy import ndimage

from oracle import klt_oracle as K

P = K.KltParams()


def _texture(W, H, shift=(0.0, 0.0), seed=3, periods=(9, 30)):
    """A smooth corner-rich analytic image sampled at pixel centres, translated by `shift`
    (content moves by +shift: value at x is the reference value at x - shift)."""
    rng = np.random.default_rng(seed)
    ys, xs = np.mgrid[0:H, 0:W].astype(np.float64) + 0.5
    xs, ys = xs - shift[0], ys - shift[1]
    img = np.zeros((H, W))
    for _ in range(6):
        th = rng.uniform(0, np.pi)
        per = rng.uniform(*periods)
        ph = rng.uniform(0, 2 * np.pi)
        img += np.sin((xs * np.cos(th) + ys * np.sin(th)) * 2 * np.pi / per + ph)
    return np.clip(np.rint(128 + 20 * img), 0, 255).astype(np.uint8)


# ---------------------------------------------------------------- Shi-Tomasi (R38)
def test_sobel_and_box_match_scipy():
    rng = np.random.default_rng(0)
    f = rng.integers(0, 256, (23, 31)).astype(np.uint8)
    Ix, Iy = K.sobel(f)
    np.testing.assert_array_equal(Ix, ndimage.sobel(f.astype(np.int64), axis=1, mode="nearest"))
    np.testing.assert_array_equal(Iy, ndimage.sobel(f.astype(np.int64), axis=0, mode="nearest"))
    a = rng.integers(-50, 50, (23, 31)).astype(np.int64)
    np.testing.assert_array_equal(K.box_sum(a, 3), ndimage.correlate(a, np.ones((3, 3), np.int64), mode="nearest"))


def test_min_eig_score_is_the_smaller_eigenvalue():
    f = _texture(40, 30)
    s = K.min_eig_score(f, 3)
    Ix, Iy = K.sobel(f)
    k = np.ones((3, 3))
    a = ndimage.correlate(Ix * Ix, k, mode="nearest")
    b = ndimage.correlate(Ix * Iy, k, mode="nearest")
    c = ndimage.correlate(Iy * Iy, k, mode="nearest")
    for y, x in [(0, 0), (5, 7), (29, 39), (15, 20), (12, 33)]:
        ev = np.linalg.eigvalsh(np.array([[a[y, x], b[y, x]], [b[y, x], c[y, x]]], np.float64))
        assert abs(float(s[y, x]) - ev[0]) <= 1e-6 * max(1.0, ev[1]), (y, x, s[y, x], ev)


def test_constant_frame_has_no_corners():
    assert K.good_features(np.full((32, 32), 77, np.uint8), P).shape == (0, 2)


def test_white_square_corners():
    """the 4 corners of a white square on black within 1.5 px."""
    f = np.zeros((64, 64), np.uint8)
    f[20:44, 16:48] = 255
    p = K.KltParams(max_corners=4, min_distance=5)
    pts = K.good_features(f, p)
    assert len(pts) == 4
    truth = [(16, 20), (47, 20), (16, 43), (47, 43)]          # corner pixels of the square
    for tx, ty in truth:
        assert min(math.hypot(x - tx, y - ty) for x, y in pts) <= 1.5, (pts, (tx, ty))


def test_greedy_selection_invariants():
    """The greedy min-distance selection is characterised by: kept corners pairwise >=
    min_distance apart; every qualifying candidate not kept lies within min_distance of a
    kept corner of higher rank; kept corners in rank order; at most max_corners."""
    f = _texture(96, 64, seed=9)
    p = K.KltParams(max_corners=25, min_distance=7.0)
    pts = K.good_features(f, p)
    s = K.min_eig_score(f, 3)
    H, W = f.shape
    thr = p.quality * float(s.max())
    rank = {}
    cand = []
    for y in range(1, H - 1):
        for x in range(1, W - 1):
            v = s[y, x]
            if v > 0 and float(v) >= thr and v >= s[y - 1:y + 2, x - 1:x + 2].max():
                cand.append((-float(v), y * W + x, x, y))
    cand.sort()
    for r, c in enumerate(cand):
        rank[(c[2], c[3])] = r
    kept = [tuple(q) for q in pts.tolist()]
    assert len(kept) <= p.max_corners
    assert [rank[q] for q in kept] == sorted(rank[q] for q in kept)
    for i, a in enumerate(kept):
        for b in kept[i + 1:]:
            assert math.dist(a, b) >= p.min_distance
    last = rank[kept[-1]]
    for c in cand[:last + 1]:
        q = (c[2], c[3])
        if q in kept:
            continue
        assert any(math.dist(q, k) < p.min_distance and rank[k] < rank[q] for k in kept), q


def test_checkerboard_min_distance():
    """checkerboard, min_dist 8 -> no two points closer than 8 px."""
    y, x = np.mgrid[0:32, 0:32]
    f = (((x // 4) + (y // 4)) % 2 * 255).astype(np.uint8)
    pts = K.good_features(f, K.KltParams(max_corners=200, min_distance=8.0))
    assert len(pts) > 4
    d = np.sqrt(((pts[:, None, :] - pts[None, :, :]) ** 2).sum(-1)) + np.eye(len(pts)) * 1e9
    assert d.min() >= 8.0


# ---------------------------------------------------------------- pyramid, bilinear (R39)
def test_pyramid_box_average():
    f = np.array([[0, 1, 2, 3], [4, 5, 6, 7], [8, 9, 10, 11], [12, 13, 14, 15], [1, 1, 1, 1]], np.uint8)
    lv = K.pyramid(f, 3, 1)
    assert [L.shape for L in lv] == [(5, 4), (2, 2), (1, 1)]
    # (0+1+4+5+2)>>2 = 3, (2+3+6+7+2)>>2 = 5, (8+9+12+13+2)>>2 = 11, (10+11+14+15+2)>>2 = 13
    assert lv[1].tolist() == [[3, 5], [11, 13]]
    assert lv[2].tolist() == [[8]]                       # (3+5+11+13+2)>>2
    assert len(K.pyramid(np.zeros((64, 48), np.uint8), 5, 20)) == 2      # 24x32, then 12x16 < 20


def test_bilinear_matches_map_coordinates():
    rng = np.random.default_rng(5)
    img = rng.uniform(0, 255, (17, 23))
    cx = rng.uniform(-3, 26, 500)
    cy = rng.uniform(-3, 20, 500)
    ref = ndimage.map_coordinates(img, [cy - 0.5, cx - 0.5], order=1, mode="nearest")
    np.testing.assert_allclose(K.bilinear(img, cx, cy), ref, atol=1e-9)
    assert K.bilinear(img, np.array([4.5]), np.array([2.5]))[0] == img[2, 4]


# ---------------------------------------------------------------- LK (R40)
def test_lk_identity():
    f = _texture(120, 90)
    pts = K.good_features(f, P)
    out, st = K.lk_track(f, f, pts, P)
    assert st.all() and len(pts) > 20
    np.testing.assert_allclose(out, pts + 0.5, atol=0.01)


@pytest.mark.parametrize("shift,tol,size,periods", [((3.0, 0.0), 0.05, (200, 150), (9, 30)),
                                                      ((1.3, -0.7), 0.05, (200, 150), (9, 30)),
                                                      ((14.0, 9.0), 0.1, (400, 300), (24, 60))])
def test_lk_recovers_known_shift(shift, tol, size, periods):
    """SPEC S:297 (+3 px within 0.5 px; here 0.05), a sub-pixel shift, and a 14 px shift
    that only the pyramid can follow with a 20-px window (4 levels at 400x300)."""
    W, H = size
    a, b = _texture(W, H, periods=periods), _texture(W, H, shift=shift, periods=periods)
    pts = K.good_features(a, P)
    pts = pts[(pts[:, 0] > 30) & (pts[:, 0] < W - 30) & (pts[:, 1] > 30) & (pts[:, 1] < H - 30)]
    out, st = K.lk_track(a, b, pts, P)
    assert st.mean() > 0.95 and len(pts) > 20
    flow = out[st] - (pts[st] + 0.5)
    assert np.abs(np.median(flow, axis=0) - np.array(shift)).max() < tol, np.median(flow, axis=0)
    assert (np.abs(flow - np.array(shift)).max(axis=1) < 0.5).mean() > 0.9


def test_lk_flat_region_is_lost():
    f = np.full((64, 64), 100, np.uint8)
    out, st = K.lk_track(f, f, np.array([[32, 32]]), P)
    assert not st[0]


# ---------------------------------------------------------------- DLT / RANSAC (R41, R42)
def _random_h(rng):
    Hm = np.eye(3) + np.array([[rng.uniform(-.05, .05), rng.uniform(-.05, .05), rng.uniform(-8, 8)],
                               [rng.uniform(-.05, .05), rng.uniform(-.05, .05), rng.uniform(-8, 8)],
                               [rng.uniform(-2e-4, 2e-4), rng.uniform(-2e-4, 2e-4), 0]])
    return Hm / Hm[2, 2]


def test_dlt_exact_cases():
    """identity within 1e-9, translation within 1e-6, a random H within 1e-6."""
    rng = np.random.default_rng(11)
    src = rng.uniform(0, 320, (4, 2))
    np.testing.assert_allclose(K.dlt(src, src), np.eye(3), atol=1e-9)
    np.testing.assert_allclose(K.dlt(src, src + [5, -2]), [[1, 0, 5], [0, 1, -2], [0, 0, 1]], atol=1e-6)
    for _ in range(5):
        Hm = _random_h(rng)
        src = rng.uniform(0, 320, (30, 2))
        np.testing.assert_allclose(K.dlt(src, K.project(Hm, src)), Hm, atol=1e-6, rtol=1e-6)
        np.testing.assert_allclose(K.minimal_homography(src[:4], K.project(Hm, src[:4])), Hm, atol=1e-6, rtol=1e-6)


def test_minimal_degenerate():
    src = np.array([[0, 0], [1, 1], [2, 2], [5, 0]], np.float64)
    assert K.minimal_homography(src, src + 1) is None


def test_splitmix64_published_values():
    """SplitMix64 (Steele, Lea & Flood 2014) from state 0: the published first outputs."""
    z, out = 0, []
    for _ in range(3):
        out.append(K.splitmix64(z))
        z = (z + 0x9E3779B97F4A7C15) & K.MASK64
    assert out == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]


def test_ransac_samples():
    n = 37
    hits = np.zeros(n)
    for it in range(2000):
        idx = K.ransac_sample(42, it, n)
        assert len(set(idx)) == 4 and all(0 <= i < n for i in idx)
        hits[idx] += 1
    assert hits.min() > 0.6 * hits.mean() and hits.max() < 1.4 * hits.mean()
    assert K.ransac_sample(42, 5, 37) == K.ransac_sample(42, 5, 37)
    assert K.ransac_sample(42, 5, 37) != K.ransac_sample(43, 5, 37)


def test_ransac_translation_no_outliers():
    rng = np.random.default_rng(2)
    src = rng.uniform(0, 300, (50, 2))
    Hm, inl, _ = K.ransac(src, src + [4.0, -1.5], P)
    assert inl.all()
    np.testing.assert_allclose(Hm, [[1, 0, 4], [0, 1, -1.5], [0, 0, 1]], atol=1e-9)


def test_ransac_with_outliers():
    """40 exact matches + 10 random outliers, thresh 3 px -> the true H within
    1e-3 and >= 40 inliers; the same seed gives the same result."""
    rng = np.random.default_rng(7)
    Hm = _random_h(rng)
    src = rng.uniform(0, 320, (50, 2))
    dst = K.project(Hm, src)
    out = rng.choice(50, 10, replace=False)
    dst[out] += rng.uniform(20, 60, (10, 2)) * rng.choice([-1, 1], (10, 2))
    H1, inl, counts = K.ransac(src, dst, P)
    assert inl.sum() >= 40 and not inl[out].any()
    np.testing.assert_allclose(H1, Hm, atol=1e-3, rtol=1e-3)
    H2, inl2, counts2 = K.ransac(src, dst, P)
    assert np.array_equal(H1, H2) and np.array_equal(inl, inl2) and np.array_equal(counts, counts2)


# ---------------------------------------------------------------- the chain
def test_chain_recovers_synthetic_homography():
    """SPEC end-to-end property: a frame pair related by a known homography (rendered
    analytically) -> the four image-corner reprojections within 1 px."""
    import synth
    cfg = synth.config("C2", T=3, S=1)
    seq = synth.generate(cfg)
    Hm, det = K.estimate(seq.frames[0, 0], seq.frames[1, 0])
    assert det["ok"] and det["inliers"].sum() >= 20
    Ht = seq.homographies[1, 0].reshape(3, 3)
    W, H = cfg.W, cfg.H
    corners = np.array([[0, 0], [W, 0], [0, H], [W, H]], np.float64)
    err = np.sqrt(((K.project(Hm.reshape(3, 3), corners) - K.project(Ht, corners)) ** 2).sum(1))
    assert err.max() < 1.0, err
