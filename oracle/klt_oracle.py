"""TEST INFRASTRUCTURE ONLY -- plain CPU oracle of the paper's motion estimation
(SURVEY.md §8(f) NEXT-4): PAPER.md App. F calls

    cv::goodFeaturesToTrack(prev, prevPts, maxCorners, qualityLevel, minDistance, ...)
    cv::calcOpticalFlowPyrLK(prev, next, prevPts, nextPts, status, err, Size(20,20), 5)
    H = cv::findHomography(prev_corner2, cur_corner2, CV_RANSAC)

(§2.4: "KLT ... is used to find feature points and the vector shifts of the pixels
... RANSAC is then used to create a homography matrix from these vectors"; §3.1.3).
This module writes those three steps out plainly in float64 NumPy, following the
algorithms in their usual order and notation (Shi & Tomasi's minimum-eigenvalue corners,
Bouguet's pyramidal Lucas-Kanade, Fischler & Bolles' RANSAC with Hartley's normalized DLT)
with the readings DESIGN.md §2 R38-R43 states where the paper (which only names OpenCV
calls) is silent.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg
may import it; the product path (paper_1702_05156_b200/) never does and shares no code.

Coordinates: pixel (x, y) covers [x, x+1) x [y, y+1) (R2); corners are returned as pixel
indices (x, y) (their centres are (x + 0.5, y + 0.5)); LK and the homography work in the
continuous coordinates of R2, so the homography estimated here is in the same convention
as the one dmsgm_step takes (R3: it maps frame-t coordinates to frame-(t-1) ones).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

MASK64 = (1 << 64) - 1


@dataclass
class KltParams:
    max_corners: int = 400        # goodFeaturesToTrack maxCorners (the paper passes a variable; R38)
    quality: float = 0.01         # qualityLevel
    min_distance: float = 10.0    # minDistance (px)
    block_size: int = 3           # structure-tensor window (OpenCV's default blockSize)
    win: int = 20                 # calcOpticalFlowPyrLK winSize: Size(20,20) (App. F)
    max_level: int = 5            # maxLevel 5 (App. F): pyramid levels 0..5
    max_iters: int = 30           # termination: 30 iterations ...
    eps: float = 0.01             # ... or a step below 0.01 px (OpenCV's default criteria)
    min_eig: float = 1e-3         # lost if lambda_min(G) / win^2 < min_eig (R40)
    ransac_iters: int = 500       # findHomography(CV_RANSAC): SPEC S:354 defaults
    ransac_thresh: float = 3.0    # reprojection threshold (px)
    seed: int = 42


# ---------------------------------------------------------------------------
# Shi-Tomasi corners (goodFeaturesToTrack), reading R38
# ---------------------------------------------------------------------------
def _pad(a, r):
    return np.pad(a, r, mode="edge")


def sobel(frame: np.ndarray):
    """3x3 Sobel derivatives of a u8 frame, replicated borders: exact integers."""
    P = _pad(frame.astype(np.int64), 1)
    H, W = frame.shape
    s = lambda dy, dx: P[1 + dy:1 + dy + H, 1 + dx:1 + dx + W]
    Ix = (s(-1, 1) + 2 * s(0, 1) + s(1, 1)) - (s(-1, -1) + 2 * s(0, -1) + s(1, -1))
    Iy = (s(1, -1) + 2 * s(1, 0) + s(1, 1)) - (s(-1, -1) + 2 * s(-1, 0) + s(-1, 1))
    return Ix, Iy


def box_sum(a: np.ndarray, block: int):
    """Sum over the block x block window centred at each pixel, replicated borders."""
    r = block // 2
    P = _pad(a, r)
    H, W = a.shape
    out = np.zeros_like(a)
    for dy in range(block):
        for dx in range(block):
            out += P[dy:dy + H, dx:dx + W]
    return out


def min_eig_score(frame: np.ndarray, block: int = 3) -> np.ndarray:
    """Shi-Tomasi score: the smaller eigenvalue of the structure tensor
    [[a, b], [b, c]] = sum over the window of [[Ix^2, IxIy], [IxIy, Iy^2]]:
    lambda_min = ((a + c) - sqrt((a - c)^2 + 4 b^2)) / 2, from the exact integer tensor in
    float64 (the discriminant is an exact integer below 2^53), rounded to float32 (the
    precision of OpenCV's eigenvalue image)."""
    Ix, Iy = sobel(frame)
    a = box_sum(Ix * Ix, block)
    b = box_sum(Ix * Iy, block)
    c = box_sum(Iy * Iy, block)
    D = (a - c) * (a - c) + 4 * b * b                    # exact int64
    lam = ((a + c).astype(np.float64) - np.sqrt(D.astype(np.float64))) * 0.5
    return lam.astype(np.float32)


def good_features(frame: np.ndarray, p: KltParams) -> np.ndarray:
    """goodFeaturesToTrack: corners as pixel indices [n][2] (x, y), in selection order.

    candidates: interior pixels (1 <= x < W-1, 1 <= y < H-1) whose score is > 0, at least
    quality x (the image's maximum score), and >= each of its 8 neighbours; visited by
    descending score, ties by ascending raster index y*W + x; a candidate is kept unless
    an already kept corner lies at distance < min_distance; at most max_corners."""
    score = min_eig_score(frame, p.block_size)
    H, W = frame.shape
    smax = float(score.max()) if score.size else 0.0
    if smax <= 0.0:
        return np.zeros((0, 2), np.int64)
    thr = p.quality * smax
    if H < 3 or W < 3:
        return np.zeros((0, 2), np.int64)
    inner = score[1:H - 1, 1:W - 1]
    ok = (inner > 0) & (inner.astype(np.float64) >= thr)
    for dy in (-1, 0, 1):                                # >= each of the 8 neighbours
        for dx in (-1, 0, 1):
            if dy or dx:
                ok &= inner >= score[1 + dy:H - 1 + dy, 1 + dx:W - 1 + dx]
    ys, xs = np.nonzero(ok)
    ys, xs = ys + 1, xs + 1
    order = np.lexsort((ys * W + xs, -score[ys, xs].astype(np.float64)))   # score desc, raster asc
    kept = []
    r2 = p.min_distance * p.min_distance
    for y, x in zip(ys[order].tolist(), xs[order].tolist()):
        if all((x - kx) ** 2 + (y - ky) ** 2 >= r2 for kx, ky in kept):
            kept.append((x, y))
            if len(kept) == p.max_corners:
                break
    return np.array(kept, np.int64).reshape(-1, 2)


# ---------------------------------------------------------------------------
# Pyramidal Lucas-Kanade (calcOpticalFlowPyrLK), reading R39 / R40
# ---------------------------------------------------------------------------
def pyramid(frame: np.ndarray, max_level: int, win: int):
    """Level 0 = the frame; level L+1 = 2x2 box average of level L, rounded half up
    ((a + b + c + d + 2) >> 2), size (w // 2, h // 2).  Levels stop before one would be
    narrower or lower than the window."""
    levels = [frame.astype(np.int64)]
    while len(levels) <= max_level:
        P = levels[-1]
        h, w = P.shape[0] // 2, P.shape[1] // 2
        if h < win or w < win:
            break
        Q = (P[0:2 * h:2, 0:2 * w:2] + P[0:2 * h:2, 1:2 * w:2] + P[1:2 * h:2, 0:2 * w:2] +
             P[1:2 * h:2, 1:2 * w:2] + 2) >> 2
        levels.append(Q)
    return [L.astype(np.float64) for L in levels]


def bilinear(img: np.ndarray, cx: np.ndarray, cy: np.ndarray) -> np.ndarray:
    """Image value at continuous coordinates (R2: pixel (i, j) centred at (i+.5, j+.5)),
    bilinear between pixel centres, border pixels repeated outside."""
    h, w = img.shape
    ux, uy = cx - 0.5, cy - 0.5
    x0, y0 = np.floor(ux), np.floor(uy)
    fx, fy = ux - x0, uy - y0
    x0, y0 = x0.astype(np.int64), y0.astype(np.int64)
    xa, xb = np.clip(x0, 0, w - 1), np.clip(x0 + 1, 0, w - 1)
    ya, yb = np.clip(y0, 0, h - 1), np.clip(y0 + 1, 0, h - 1)
    top = img[ya, xa] * (1 - fx) + img[ya, xb] * fx
    bot = img[yb, xa] * (1 - fx) + img[yb, xb] * fx
    return top * (1 - fy) + bot * fy


def lk_track(prev: np.ndarray, nxt: np.ndarray, pts: np.ndarray, p: KltParams):
    """Track corner pixel indices pts [n][2] from prev to next.  Returns (next points in
    continuous coordinates [n][2] float64, status [n] bool).

    Per point c (continuous, = index + 0.5), coarsest level first, guess g = 0:
      p_L = c / 2^L; window samples s = p_L + (i - (win-1)/2, j - (win-1)/2), i, j < win;
      I = prev_L(s) bilinear, Ix = (I(s + e_x) - I(s - e_x)) / 2, Iy likewise;
      G = sum [[Ix^2, IxIy], [IxIy, Iy^2]]; lost if lambda_min(G) / win^2 < min_eig;
      v = 0; up to max_iters times: e = I(s) - next_L(s + g + v), b = sum [e Ix, e Iy],
      d = G^-1 b, v += d, stop when |d| < eps; lost if p_L + g + v leaves the level image;
      g <- 2 (g + v) for the next finer level.  Result c + g_0 + v_0."""
    P, Q = pyramid(prev, p.max_level, p.win), pyramid(nxt, p.max_level, p.win)
    nlev = len(P)
    off = np.arange(p.win, dtype=np.float64) - (p.win - 1) / 2.0
    ox, oy = np.meshgrid(off, off)
    out = np.zeros((len(pts), 2))
    status = np.ones(len(pts), bool)
    for k, (x, y) in enumerate(pts):
        c = np.array([x + 0.5, y + 0.5])
        g = np.zeros(2)
        for L in range(nlev - 1, -1, -1):
            pl = c / (2 ** L)
            sx, sy = pl[0] + ox, pl[1] + oy
            I = bilinear(P[L], sx, sy)
            Ix = (bilinear(P[L], sx + 1, sy) - bilinear(P[L], sx - 1, sy)) / 2
            Iy = (bilinear(P[L], sx, sy + 1) - bilinear(P[L], sx, sy - 1)) / 2
            gxx, gxy, gyy = (Ix * Ix).sum(), (Ix * Iy).sum(), (Iy * Iy).sum()
            lam = ((gxx + gyy) - np.sqrt((gxx - gyy) ** 2 + 4 * gxy * gxy)) / 2
            det = gxx * gyy - gxy * gxy
            v = np.zeros(2)
            if lam / (p.win * p.win) < p.min_eig or det <= 0:
                if L == 0:                       # too little texture: lost
                    status[k] = False
                    break
                g = 2 * g                        # a coarse level without texture: skipped
                continue
            h, w = P[L].shape
            for _ in range(p.max_iters):
                e = I - bilinear(Q[L], sx + g[0] + v[0], sy + g[1] + v[1])
                bx, by = (e * Ix).sum(), (e * Iy).sum()
                d = np.array([gyy * bx - gxy * by, gxx * by - gxy * bx]) / det
                v = v + d
                q = pl + g + v
                if L == 0 and not (0 <= q[0] < w and 0 <= q[1] < h):
                    status[k] = False            # the point left the frame
                    break
                if d[0] * d[0] + d[1] * d[1] < p.eps * p.eps:
                    break
            if not status[k]:
                break
            g = 2 * (g + v) if L > 0 else g + v
        out[k] = c + g if status[k] else np.nan
    return out, status


# ---------------------------------------------------------------------------
# Normalized DLT and RANSAC (findHomography(CV_RANSAC)), readings R41 / R42
# ---------------------------------------------------------------------------
def hartley(pts: np.ndarray):
    """Similarity T moving the centroid to 0 and the mean distance to sqrt(2)."""
    cen = pts.mean(axis=0)
    d = np.sqrt(((pts - cen) ** 2).sum(axis=1)).mean()
    s = np.sqrt(2.0) / d if d > 0 else 1.0
    return np.array([[s, 0, -s * cen[0]], [0, s, -s * cen[1]], [0, 0, 1.0]])


def dlt(src: np.ndarray, dst: np.ndarray) -> np.ndarray:
    """Normalized DLT (Hartley): H (3x3, H[2,2] = 1) minimising the algebraic error of
    dst ~ H src over >= 4 correspondences: the right singular vector of the smallest
    singular value of the 2n x 9 system in Hartley-normalized coordinates, denormalized."""
    Ts, Td = hartley(src), hartley(dst)
    s = (Ts @ np.c_[src, np.ones(len(src))].T).T
    d = (Td @ np.c_[dst, np.ones(len(dst))].T).T
    A = []
    for (x, y, _), (u, v, _) in zip(s, d):
        A.append([0, 0, 0, -x, -y, -1, v * x, v * y, v])
        A.append([x, y, 1, 0, 0, 0, -u * x, -u * y, -u])
    _, _, Vt = np.linalg.svd(np.array(A))
    Hn = Vt[-1].reshape(3, 3)
    Hm = np.linalg.inv(Td) @ Hn @ Ts
    return Hm / Hm[2, 2]


def project(Hm: np.ndarray, pts: np.ndarray) -> np.ndarray:
    q = (Hm @ np.c_[pts, np.ones(len(pts))].T).T
    return q[:, :2] / q[:, 2:3]


def splitmix64(z: int) -> int:
    """The SplitMix64 output function (Steele, Lea & Flood 2014) of a 64-bit state."""
    z = (z + 0x9E3779B97F4A7C15) & MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def ransac_sample(seed: int, it: int, n: int):
    """R42: the 4 distinct match indices of RANSAC iteration `it` (counter-based, so both
    sides draw the same sets): draw k = 0, 1, ... gives floor(hi32(splitmix64(state)) * n
    / 2^32) with state = seed * 2^32 + it * 64 + k; repeats are skipped; None if 64 draws
    do not give 4 distinct indices."""
    got = []
    for k in range(64):
        z = splitmix64(((seed << 32) + it * 64 + k) & MASK64)
        i = ((z >> 32) * n) >> 32
        if i not in got:
            got.append(i)
            if len(got) == 4:
                return got
    return None


def _collinear(pts: np.ndarray) -> bool:
    """Any 3 of the 4 points collinear: |cross| <= 1e-6 x (squared extent)."""
    ext = max(np.ptp(pts[:, 0]), np.ptp(pts[:, 1]), 1e-12)
    for a in range(4):
        for b in range(a + 1, 4):
            for c in range(b + 1, 4):
                u, v = pts[b] - pts[a], pts[c] - pts[a]
                if abs(u[0] * v[1] - u[1] * v[0]) <= 1e-6 * ext * ext:
                    return True
    return False


def minimal_homography(src4: np.ndarray, dst4: np.ndarray):
    """The homography with H[2,2] = 1 through 4 correspondences (8x8 linear system), or
    None for a degenerate sample (3 collinear points in either set)."""
    if _collinear(src4) or _collinear(dst4):
        return None
    A = np.zeros((8, 8))
    r = np.zeros(8)
    for i, ((x, y), (u, v)) in enumerate(zip(src4, dst4)):
        A[2 * i] = [x, y, 1, 0, 0, 0, -u * x, -u * y]
        A[2 * i + 1] = [0, 0, 0, x, y, 1, -v * x, -v * y]
        r[2 * i], r[2 * i + 1] = u, v
    try:
        h = np.linalg.solve(A, r)
    except np.linalg.LinAlgError:
        return None
    return np.append(h, 1.0).reshape(3, 3)


def ransac(src: np.ndarray, dst: np.ndarray, p: KltParams):
    """RANSAC (Fischler & Bolles): for each iteration a minimal 4-point model; inliers
    are the matches with squared reprojection error ||H src - dst||^2 < thresh^2; the
    model with the most inliers wins (ties: the earliest iteration); the result is the
    normalized DLT over the winner's inliers.  Returns (H or None, inlier mask, counts per
    iteration)."""
    n = len(src)
    counts = np.full(p.ransac_iters, -1, np.int64)
    if n < 4:
        return None, np.zeros(n, bool), counts
    best, best_it, best_mask = -1, -1, None
    t2 = p.ransac_thresh * p.ransac_thresh
    for it in range(p.ransac_iters):
        idx = ransac_sample(p.seed, it, n)
        if idx is None:
            continue
        Hm = minimal_homography(src[idx], dst[idx])
        if Hm is None:
            continue
        err = ((project(Hm, src) - dst) ** 2).sum(axis=1)
        mask = err < t2
        counts[it] = int(mask.sum())
        if counts[it] > best:
            best, best_it, best_mask = counts[it], it, mask
    if best < 4:
        return None, np.zeros(n, bool), counts
    return dlt(src[best_mask], dst[best_mask]), best_mask, counts


# ---------------------------------------------------------------------------
# the whole chain for one frame pair
# ---------------------------------------------------------------------------
def estimate(prev: np.ndarray, nxt: np.ndarray, p: KltParams = None):
    """App. F's chain for frames t-1 (prev) and t (next): corners on prev, LK to next,
    tracked pairs -> RANSAC.  Returns (H_t [9] mapping frame-t continuous coordinates to
    frame-(t-1) ones (R3) -- identity when estimation fails --, details dict)."""
    p = p or KltParams()
    pts = good_features(prev, p)
    nxt_pts, st = lk_track(prev, nxt, pts, p)
    src = nxt_pts[st]                                   # frame t
    dst = pts[st].astype(np.float64) + 0.5              # frame t-1 (pixel centres)
    Hm, inl, counts = ransac(src, dst, p)
    ok = Hm is not None
    return (Hm if ok else np.eye(3)).reshape(9), dict(corners=pts, tracked=nxt_pts, status=st, inliers=inl,
                                                      counts=counts, ok=ok)
