"""Pins for the CPU oracle.

Each test checks the oracle against something other than itself: values worked
by hand from the paper's equations (tests/golden/), closed forms, brute-force
geometry, or invariants that the paper fixes.  No expected value here comes from
the CUDA path or from re-running the oracle's own formula.
"""
import math
import os

import numpy as np
import pytest
import yaml

import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
IDENT = np.eye(3).reshape(9)


def _params(oracle_mod, **kw):
    base = dict(theta_s=4.0, theta_d=4.0, var_init=255.0, age_cap=30.0, var_floor_match=0.1,
                var_floor_classify=0.25, decay_lambda=0.0, decay_var_thresh=2500.0, num_streams=1)
    base.update(kw)
    return oracle_mod.OracleParams(**base)


def _state_from(Hb, Wb, A, C):
    st = np.empty((6, Hb, Wb), np.float32)
    for i in range(3):
        st[i] = A[i]
        st[3 + i] = C[i]
    return st


def _one_step(oracle_mod, frame, state, N, H=IDENT, **kw):
    Hh, W = frame.shape
    o = oracle_mod.Oracle(W, Hh, N, _params(oracle_mod, **kw))
    o.set_state(0, state)
    mask = o.step(frame[None], np.asarray(H, np.float64).reshape(1, 9))[0]
    out = o.get_state(0)
    o.close()
    return out, mask


def _ulps(a, b):
    a = np.float32(a)
    b = np.float32(b)
    return abs(int(a.view(np.int32)) - int(b.view(np.int32)))


# --------------------------------------------------------------------------
# P1-P5 + per-pixel + cap: hand-worked single-block updates (tests/golden)
# --------------------------------------------------------------------------
with open(os.path.join(GOLDEN, "dsgm_hand_worked.yaml")) as f:
    _CASES = yaml.safe_load(f)["cases"]


@pytest.mark.parametrize("case", _CASES, ids=[c["id"] for c in _CASES])
def test_hand_worked(oracle_mod, case):
    N = case["N"]
    frame = np.array(case["pixels"], np.uint8)
    assert frame.shape == (N, N)
    st = _state_from(1, 1, case["A"], case["C"])
    out, mask = _one_step(oracle_mod, frame, st, N, theta_s=case["theta_s"])
    for i in range(3):
        assert _ulps(out[i, 0, 0], case["expect_A"][i]) <= 2, (case["id"], "A", i, out[:, 0, 0])
        assert _ulps(out[3 + i, 0, 0], case["expect_C"][i]) <= 2, (case["id"], "C", i, out[:, 0, 0])
    assert np.all(mask == case["expect_mask"]), (case["id"], mask)


# --------------------------------------------------------------------------
# First frame (R8): A = C = (M, var_init, 1), classified normally
# --------------------------------------------------------------------------
def test_first_frame_init(oracle_mod):
    rng = np.random.default_rng(0)
    N = 4
    frame = rng.integers(0, 256, (8, 12), dtype=np.uint8)
    o = oracle_mod.Oracle(12, 8, N, _params(oracle_mod))
    mask = o.step(frame[None], IDENT[None])[0]
    st = o.get_state(0)
    M = frame.reshape(2, N, 3, N).astype(np.float64).mean(axis=(1, 3))
    np.testing.assert_array_equal(st[0], M.astype(np.float32))
    np.testing.assert_array_equal(st[3], M.astype(np.float32))
    assert np.all(st[1] == 255) and np.all(st[4] == 255)
    assert np.all(st[2] == 1) and np.all(st[5] == 1)
    # classification against (M, 255): fg iff (I-M)^2 > 4*255 (App. E, R14)
    Mpx = np.kron(M, np.ones((N, N)))
    expect = np.where((frame - Mpx) ** 2 > 1020.0, 255, 0)
    np.testing.assert_array_equal(mask, expect)


# --------------------------------------------------------------------------
# P6: identity H makes S1-S3 the identity map on the state (bitwise)
# --------------------------------------------------------------------------
@pytest.mark.parametrize("N", [1, 2, 4, 8, 16])
def test_identity_weights(oracle_mod, N):
    for (W, H) in [(64, 48), (320, 240), (1920, 1088), (3840, 2160)]:
        if W % N or H % N:
            continue
        Wb, Hb = W // N, H // N
        for bi in sorted({0, 1, Wb // 2, Wb - 1}):
            for bj in sorted({0, Hb // 3, Hb - 1}):
                exp, src, w, sw = oracle_mod.mix_weights(W, H, N, IDENT, bi, bj)
                assert not exp
                assert src[0] == (bi, bj)
                assert w.tolist() == [1.0, 0.0, 0.0, 0.0] and sw == 1.0


def _probe_tilde_A(oracle_mod, state, H, N, W, Hh, **kw):
    """theta_s -> 0: nothing matches, so A after the step equals the tilde A (R11)."""
    frame = np.full((Hh, W), 7, np.uint8)
    out, _ = _one_step(oracle_mod, frame, state, N, H, theta_s=1e-30, **kw)
    return out[0:3], out


@pytest.mark.parametrize("lam", [0.0, 0.001])
def test_identity_tilde_is_previous_state(oracle_mod, lam):
    rng = np.random.default_rng(1)
    N, W, Hh = 4, 40, 24
    st = synth.random_state(rng, Hh // N, W // N, var_max=2400.0)  # all var <= theta_v
    st[0][st[0] == 7.0] = 8.0  # avoid an exact M == mu match
    A, _ = _probe_tilde_A(oracle_mod, st, IDENT, N, W, Hh, decay_lambda=lam)
    np.testing.assert_array_equal(A, st[0:3])


# --------------------------------------------------------------------------
# P7: always-match running-mean closed form
# --------------------------------------------------------------------------
def test_running_mean_closed_form(oracle_mod):
    rng = np.random.default_rng(2)
    N, T = 4, 29
    blocks = rng.integers(0, 256, (T, N, N)).astype(np.uint8)
    o = oracle_mod.Oracle(N, N, N, _params(oracle_mod, theta_s=1e9))
    mus, Vs = [], []
    for t in range(T):
        o.step(blocks[t][None], IDENT[None])
        st = o.get_state(0)
        I = blocks[: t + 1].astype(np.float64)
        mu_t = I.mean(axis=(1, 2)).mean()               # mean of block means (Eq. 3 unrolled)
        mus.append(mu_t)
        if t >= 1:
            Vs.append(np.max((mu_t - blocks[t].astype(np.float64)) ** 2))   # Eq. 6
        var_t = (255.0 + sum(Vs)) / (t + 1)            # Eq. 5 unrolled
        assert abs(st[0, 0, 0] - mu_t) <= 2e-5 * max(1.0, abs(mu_t)), t
        assert abs(st[1, 0, 0] - var_t) <= 1e-4 * max(1.0, var_t), (t, st[1, 0, 0], var_t)
        assert st[2, 0, 0] == min(t + 1, 30)            # Eq. 7 + cap
    o.close()


# --------------------------------------------------------------------------
# P8 / P9: step change background -> foreground under identity H
# --------------------------------------------------------------------------
@pytest.mark.parametrize("t0,expect_fg", [(1, 1), (5, 5), (10, 10), (29, 29), (30, None), (40, None)])
def test_step_change(oracle_mod, t0, expect_fg):
    N = 4
    o = oracle_mod.Oracle(8, 8, N, _params(oracle_mod, decay_lambda=0.001))
    fg_frames = []
    T = t0 + 70
    for t in range(T):
        v = 50 if t < t0 else 150
        m = o.step(np.full((1, 8, 8), v, np.uint8), IDENT[None])
        assert np.all(m == m.flat[0])
        if m.flat[0] == 255:
            fg_frames.append(t)
    if expect_fg is None:
        # P9: alpha_A = cap and the candidate caps at 30 too; Eq. 10 is strict -> never swaps
        assert fg_frames == list(range(t0, T))
    else:
        # P8: the candidate overtakes after exactly alpha_A = min(t0, 30) frames
        assert fg_frames == list(range(t0, t0 + expect_fg))
    o.close()


# --------------------------------------------------------------------------
# P10: translation by whole blocks is an index shift; exposed strip is FRESH
# --------------------------------------------------------------------------
@pytest.mark.parametrize("k,l", [(1, 0), (0, -2), (-3, 1), (2, 2)])
def test_block_translation(oracle_mod, k, l):
    rng = np.random.default_rng(3)
    N, W, Hh = 4, 48, 32
    Wb, Hb = W // N, Hh // N
    st = synth.random_state(rng, Hb, Wb, var_max=2400.0)
    H = np.array([1.0, 0.0, k * N, 0.0, 1.0, l * N, 0.0, 0.0, 1.0])
    A, out = _probe_tilde_A(oracle_mod, st, H, N, W, Hh)
    for bj in range(Hb):
        for bi in range(Wb):
            sx, sy = bi + k, bj + l
            if 0 <= sx < Wb and 0 <= sy < Hb:
                assert np.array_equal(A[:, bj, bi], st[0:3, sy, sx])
            else:
                assert A[:, bj, bi].tolist() == [7.0, 255.0, 1.0]
                assert out[3:6, bj, bi].tolist() == [7.0, 255.0, 1.0]


# --------------------------------------------------------------------------
# P11: half-block translation: closed-form two-source mixture
# --------------------------------------------------------------------------
def test_half_block_translation(oracle_mod):
    N, W, Hh = 4, 16, 4
    st = np.zeros((6, 1, 4), np.float32)
    st[0, 0] = [120.0, 100.0, 60.0, 10.0]
    st[1, 0] = [20.0, 10.0, 1.0, 3.0]
    st[2, 0] = [20.0, 10.0, 30.0, 2.0]
    st[3:6] = st[0:3]
    H = np.array([1.0, 0.0, N / 2.0, 0.0, 1.0, 0.0, 0.0, 0.0, 1.0])
    A, _ = _probe_tilde_A(oracle_mod, st, H, N, W, Hh)
    # (120,20,20) & (100,10,10) -> (110, 15 + 10^2, 15)   (R6 mixture)
    assert A[:, 0, 0].tolist() == [110.0, 115.0, 15.0]
    assert A[:, 0, 1].tolist() == [80.0, 5.5 + 400.0, 20.0]
    assert A[:, 0, 2].tolist() == [35.0, 2.0 + 625.0, 16.0]
    # last column: its right neighbour is out of range -> only itself, renormalised (R5)
    assert A[:, 0, 3].tolist() == [10.0, 3.0, 2.0]


# --------------------------------------------------------------------------
# P12: weights equal brute-force polygon overlap areas
# --------------------------------------------------------------------------
def _clip(poly, x0, x1, y0, y1):
    """Sutherland-Hodgman clip of a polygon against an axis-aligned rectangle."""
    def clip_edge(pts, inside, inter):
        out = []
        for i in range(len(pts)):
            cur, prev = pts[i], pts[i - 1]
            if inside(cur):
                if not inside(prev):
                    out.append(inter(prev, cur))
                out.append(cur)
            elif inside(prev):
                out.append(inter(prev, cur))
        return out

    def ix(x):
        return lambda p, q: (x, p[1] + (q[1] - p[1]) * (x - p[0]) / (q[0] - p[0]))

    def iy(y):
        return lambda p, q: (p[0] + (q[0] - p[0]) * (y - p[1]) / (q[1] - p[1]), y)

    pts = list(poly)
    for inside, inter in ((lambda p: p[0] >= x0, ix(x0)), (lambda p: p[0] <= x1, ix(x1)),
                          (lambda p: p[1] >= y0, iy(y0)), (lambda p: p[1] <= y1, iy(y1))):
        pts = clip_edge(pts, inside, inter)
        if not pts:
            return []
    return pts


def _area(pts):
    if len(pts) < 3:
        return 0.0
    s = 0.0
    for i in range(len(pts)):
        x1, y1 = pts[i - 1]
        x2, y2 = pts[i]
        s += x1 * y2 - x2 * y1
    return abs(s) / 2.0


def _overlaps(poly, Wb, Hb):
    xs = [p[0] for p in poly]
    ys = [p[1] for p in poly]
    res = {}
    for cy in range(math.floor(min(ys)) - 1, math.floor(max(ys)) + 2):
        for cx in range(math.floor(min(xs)) - 1, math.floor(max(xs)) + 2):
            a = _area(_clip(poly, cx, cx + 1, cy, cy + 1))
            if a > 1e-15 and 0 <= cx < Wb and 0 <= cy < Hb:
                res[(cx, cy)] = a
    return res


def _apply(h, x, y):
    w = h[6] * x + h[7] * y + h[8]
    return (h[0] * x + h[1] * y + h[2]) / w, (h[3] * x + h[4] * y + h[5]) / w


@pytest.mark.parametrize("N", [1, 4, 8])
def test_weights_equal_polygon_overlap(oracle_mod, N):
    rng = np.random.default_rng(4 + N)
    W, Hh = 160, 96
    Wb, Hb = W // N, Hh // N
    checked = 0
    for trial in range(300):
        h = synth.random_homography(rng, W, Hh, shift=6.0 * N, rot_deg=0.3, zoom=0.005, persp=2e-5)
        bi, bj = int(rng.integers(0, Wb)), int(rng.integers(0, Hb))
        exposed, src, w, sw = oracle_mod.mix_weights(W, Hh, N, h, bi, bj)
        cx, cy = _apply(h, N * bi + N / 2.0, N * bj + N / 2.0)
        u, v = cx / N, cy / N
        # R4 footprint: unit square (in block units) centred at H(c)/N
        sq = [(u - 0.5, v - 0.5), (u + 0.5, v - 0.5), (u + 0.5, v + 0.5), (u - 0.5, v + 0.5)]
        ref = _overlaps(sq, Wb, Hb)
        if not ref:
            assert exposed
            continue
        assert not exposed
        got = {src[k]: float(w[k]) for k in range(4) if w[k] != 0.0}
        assert set(got) == set(ref), (got, ref)
        for key in ref:
            assert abs(got[key] - ref[key]) < 2e-6, (key, got[key], ref[key])
        assert abs(sw - sum(ref.values())) < 4e-6
        checked += 1
    assert checked > 150


@pytest.mark.parametrize("W,Hh,N", [(1920, 1080, 4), (3840, 2160, 8), (1920, 1080, 1)])
def test_weights_equal_polygon_overlap_full_size(oracle_mod, W, Hh, N):
    """P12 at the C4 / C5 / C4p frame coordinates (up to 3840 px), with perspective terms:
    the fp32 displacement-form projection (R17) keeps the overlap areas within 2e-6 of the
    fp64 polygon clip even where the coordinates themselves are ~4e3 (an fp32 ulp of a
    coordinate there is 2.4e-4 px)."""
    rng = np.random.default_rng(1080 + N)
    Wb, Hb = W // N, Hh // N
    checked = 0
    worst = 0.0
    for trial in range(400):
        h = synth.random_homography(rng, W, Hh, shift=4.0 * N, rot_deg=0.05, zoom=0.0005, persp=2e-6)
        # blocks anywhere, with a third of them in the corners where coordinates are largest
        if trial % 3 == 0:
            bi = int(rng.choice([rng.integers(0, 4), rng.integers(Wb - 4, Wb)]))
            bj = int(rng.choice([rng.integers(0, 4), rng.integers(Hb - 4, Hb)]))
        else:
            bi, bj = int(rng.integers(0, Wb)), int(rng.integers(0, Hb))
        exposed, src, w, sw = oracle_mod.mix_weights(W, Hh, N, h, bi, bj)
        cx, cy = _apply(h, N * bi + N / 2.0, N * bj + N / 2.0)
        u, v = cx / N, cy / N
        sq = [(u - 0.5, v - 0.5), (u + 0.5, v - 0.5), (u + 0.5, v + 0.5), (u - 0.5, v + 0.5)]
        ref = _overlaps(sq, Wb, Hb)
        if not ref:
            assert exposed
            continue
        assert not exposed
        got = {src[k]: float(w[k]) for k in range(4) if w[k] != 0.0}
        ref = {k: a for k, a in ref.items() if a > 2e-6 or k in got}
        assert set(got) <= set(_overlaps(sq, Wb, Hb)) and set(ref) <= set(got), (got, ref)
        for key in ref:
            worst = max(worst, abs(got[key] - ref[key]))
        checked += 1
    print(f"P12 {W}x{Hh} N={N}: worst |area error| {worst:.2e} over {checked} blocks")
    assert worst < 2e-6, worst
    assert checked > 300


@pytest.mark.parametrize("N", [2, 4, 8])
def test_translation_quad_equals_square(oracle_mod, N):
    """For a pure translation the true warped block (a quad) IS the square footprint."""
    rng = np.random.default_rng(40 + N)
    W, Hh = 128, 64
    Wb, Hb = W // N, Hh // N
    for trial in range(200):
        tx, ty = rng.uniform(-3 * N, 3 * N, 2)
        h = np.array([1.0, 0.0, tx, 0.0, 1.0, ty, 0.0, 0.0, 1.0])
        bi, bj = int(rng.integers(0, Wb)), int(rng.integers(0, Hb))
        corners = [(N * bi, N * bj), (N * bi + N, N * bj), (N * bi + N, N * bj + N), (N * bi, N * bj + N)]
        quad = [tuple(c / N for c in _apply(h, x, y)) for (x, y) in corners]
        ref = _overlaps(quad, Wb, Hb)
        exposed, src, w, sw = oracle_mod.mix_weights(W, Hh, N, h, bi, bj)
        if not ref:
            assert exposed
            continue
        got = {src[k]: float(w[k]) for k in range(4) if w[k] != 0.0}
        assert set(got) == set(ref)
        for key in ref:
            assert abs(got[key] - ref[key]) < 2e-6


def test_weights_vs_true_quad_small_motion(oracle_mod):
    """R4 approximation bound: with <=0.05 deg rotation and 0.05% zoom (the C4 recipe),
    the square footprint's areas stay within 1e-2 of the true warped quad's areas."""
    rng = np.random.default_rng(77)
    N, W, Hh = 4, 1920, 1080
    Wb, Hb = W // N, Hh // N
    worst = 0.0
    for trial in range(200):
        h = synth.random_homography(rng, W, Hh, shift=2.0, rot_deg=0.05, zoom=0.0005, persp=0.0)
        bi, bj = int(rng.integers(1, Wb - 1)), int(rng.integers(1, Hb - 1))
        corners = [(N * bi, N * bj), (N * bi + N, N * bj), (N * bi + N, N * bj + N), (N * bi, N * bj + N)]
        quad = [tuple(c / N for c in _apply(h, x, y)) for (x, y) in corners]
        ref = _overlaps(quad, Wb, Hb)
        exposed, src, w, sw = oracle_mod.mix_weights(W, Hh, N, h, bi, bj)
        got = {src[k]: float(w[k]) for k in range(4) if w[k] != 0.0}
        for key in set(ref) | set(got):
            worst = max(worst, abs(got.get(key, 0.0) - ref.get(key, 0.0)))
    assert worst < 1e-2, worst


# --------------------------------------------------------------------------
# classification boundary (App. E P:657 uses <= for background)
# --------------------------------------------------------------------------
def test_classify_boundary(oracle_mod):
    N = 4
    frame = np.array([[110, 111, 90, 89], [100, 100, 100, 100], [0, 255, 120, 80], [100, 100, 100, 100]], np.uint8)
    st = _state_from(1, 1, [100.0, 25.0, 5.0], [3.0, 1.0, 1.0])   # T = 4*25 = 100
    out, mask = _one_step(oracle_mod, frame, st, N, theta_s=1e-30)
    assert out[0:3, 0, 0].tolist() == [100.0, 25.0, 5.0]
    expect = np.where((frame.astype(np.int64) - 100) ** 2 > 100, 255, 0)
    assert expect[0].tolist() == [0, 255, 0, 255]
    np.testing.assert_array_equal(mask, expect)


def test_classify_floor(oracle_mod):
    """var_A below f_c = 0.25 uses the floor: (I-mu)^2 = 1 > 4*0.25 is NOT > 1 -> background."""
    N = 2
    frame = np.array([[101, 99], [102, 100]], np.uint8)
    st = _state_from(1, 1, [100.0, 0.0, 5.0], [3.0, 1.0, 1.0])
    _, mask = _one_step(oracle_mod, frame, st, N, theta_s=1e-30)
    assert mask.tolist() == [[0, 0], [255, 0]]


# --------------------------------------------------------------------------
# P14: age decay closed form
# --------------------------------------------------------------------------
def test_decay_closed_form(oracle_mod):
    N = 2
    st = _state_from(1, 1, [100.0, 3500.0, 10.0], [3.0, 1.0, 1.0])
    A, _ = _probe_tilde_A(oracle_mod, st, IDENT, N, N, N, decay_lambda=0.001, decay_var_thresh=2500.0)
    # lambda is the fp32 0.001, so x = 1.0000000475; within 1 ulp (R18; the plain form's
    # comparison is tests/test_oracle_forms.py::test_p14_decay_within_one_ulp_of_plain)
    assert _ulps(A[2, 0, 0], np.float32(10.0) * np.float32(math.exp(-float(np.float32(0.001)) * 1000.0))) <= 1
    assert A[1, 0, 0] == 3500.0 and A[0, 0, 0] == 100.0
    # at or below the threshold: no decay
    st = _state_from(1, 1, [100.0, 2500.0, 10.0], [3.0, 1.0, 1.0])
    A, _ = _probe_tilde_A(oracle_mod, st, IDENT, N, N, N, decay_lambda=0.001, decay_var_thresh=2500.0)
    assert A[2, 0, 0] == 10.0


# --------------------------------------------------------------------------
# exposure (R5/R8): w <= 0 and far-out projections reset the block
# --------------------------------------------------------------------------
def test_exposure(oracle_mod):
    N, W, Hh = 4, 16, 16
    for H in (np.array([1, 0, 0, 0, 1, 0, 0, 0, -1.0]),            # w < 0
              np.array([1, 0, 1e6, 0, 1, 0, 0, 0, 1.0]),           # far out
              np.array([1, 0, 0, 0, 1, 0, 1.0, 0, -1000.0])):      # w <= 0 on part of the image
        exposed_any = False
        for bi in range(W // N):
            for bj in range(Hh // N):
                e, *_ = oracle_mod.mix_weights(W, Hh, N, H, bi, bj)
                exposed_any |= e
        assert exposed_any
    # R5: a projective scale outside (2^-100, 2^100) is degenerate: every block is exposed
    for H in (np.array([1, 0, 0, 0, 1, 0, 0, 0, 1e31]),           # w = 1e31 everywhere
              np.array([1, 0, 0, 0, 1, 0, 0, 0, 1e-31])):         # w = 1e-31 everywhere (px = 0 for no block)
        for bi in range(W // N):
            for bj in range(Hh // N):
                e, *_ = oracle_mod.mix_weights(W, Hh, N, H, bi, bj)
                assert e, (H, bi, bj)


# --------------------------------------------------------------------------
# invariants over a whole synthetic sequence (north_star / SPEC S:230-235)
# --------------------------------------------------------------------------
def test_sequence_invariants(oracle_mod):
    seq = synth.generate(synth.config("C2", T=40))
    p = _params(oracle_mod, decay_lambda=0.001)
    o = oracle_mod.Oracle(320, 240, 4, p)
    prev = None
    for t in range(40):
        m = o.step(seq.frames[t], seq.homographies[t])
        st = o.get_state(0)
        assert set(np.unique(m).tolist()) <= {0, 255}
        assert np.all(np.isfinite(st))
        assert np.all((st[2] > 0) & (st[2] <= 30)) and np.all((st[5] > 0) & (st[5] <= 30))
        assert np.all(st[1] >= 0) and np.all(st[4] >= 0)
        assert np.all((st[0] >= 0) & (st[0] <= 255.0001)) and np.all((st[3] >= 0) & (st[3] <= 255.0001))
        # after S7 the candidate never has a strictly larger age than the apparent model
        assert np.all(st[5] <= st[2])
        prev = st
    assert prev is not None
    o.close()


def test_integer_age_regime(oracle_mod):
    """Identity H, lambda=0: ages stay integers and alpha_A >= alpha_C (R19)."""
    rng = np.random.default_rng(9)
    N, W, Hh = 2, 32, 16
    o = oracle_mod.Oracle(W, Hh, N, _params(oracle_mod))
    base = rng.integers(40, 200, (Hh, W))
    for t in range(60):
        fr = np.clip(base + rng.normal(0, 3, base.shape) + (80 if (t // 15) % 2 else 0), 0, 255).astype(np.uint8)
        o.step(fr[None], IDENT[None])
        st = o.get_state(0)
        assert np.all(st[2] == np.rint(st[2])) and np.all(st[5] == np.rint(st[5]))
        assert np.all(st[2] >= st[5])
    o.close()


# --------------------------------------------------------------------------
# quality sanity: per-pixel moving square
# --------------------------------------------------------------------------
def test_moving_square_quality(oracle_mod):
    cfg = synth.config("C1", N=1)
    seq = synth.generate(cfg, with_gt=True)
    masks, _, _ = oracle_mod.run_sequence(seq.frames, seq.homographies, 1, _params(oracle_mod))
    for t in range(3, cfg.T):
        g = seq.gt[t, 0] > 0
        m = masks[t, 0] > 0
        assert (m & g).sum() / g.sum() >= 0.9
        assert (m & ~g).sum() / (~g).sum() < 0.02


# --------------------------------------------------------------------------
# App. E compat rules (R27/R28): hand-worked
# --------------------------------------------------------------------------
def test_appendix_update_rule(oracle_mod):
    # App. E: alpha = 1/age (before the increment): age 4, I=120, mu=100, var=255
    N = 1
    st = _state_from(1, 1, [100.0, 255.0, 4.0], [0.0, 255.0, 1.0])
    out, _ = _one_step(oracle_mod, np.array([[120]], np.uint8), st, N, update_rule=1)
    # mu = 0.75*100 + 0.25*120 = 105; V = 225; var = 0.75*255 + 0.25*225 = 247.5; age 5
    assert out[0:3, 0, 0].tolist() == [105.0, 247.5, 5.0]
    # R22 for both rules: a fractional age near the cap (after mixing / decay, R19) is capped,
    # min(age~ + 1, 30) -- not App. E's integer `if (age < AGE_THRESH) age++`, which would
    # give 30.5 and break 1 <= age <= cap; alpha = 1/29.5
    for form in (0, 1):
        st = _state_from(1, 1, [100.0, 255.0, 29.5], [0.0, 255.0, 1.0])
        out, _ = _one_step(oracle_mod, np.array([[100]], np.uint8), st, N, update_rule=1, form=form)
        assert out[2, 0, 0] == 30.0 and out[0, 0, 0] == 100.0
        out, _ = _one_step(oracle_mod, np.array([[100]], np.uint8), st, N, update_rule=0, form=form)
        assert out[2, 0, 0] == 30.0


def test_appendix_classify_rule(oracle_mod):
    # App. E: background iff (mu_A - I)^2 <= THETA_D * max(0.25, I)
    N = 2
    frame = np.array([[20, 21], [4, 0]], np.uint8)
    st = _state_from(1, 1, [2.0, 1000.0, 5.0], [200.0, 1.0, 1.0])
    _, mask = _one_step(oracle_mod, frame, st, N, theta_s=1e-30, classify_rule=1)
    # 18^2=324 > 80 fg; 19^2=361 > 84 fg; 2^2=4 <= 16 bg; 2^2=4 > 4*0.25=1 fg
    assert mask.tolist() == [[255, 255], [0, 255]]


# --------------------------------------------------------------------------
# R6: renormalisation only when the footprint is clipped by the grid border
# --------------------------------------------------------------------------
def test_clipped_renormalisation(oracle_mod):
    N, W, Hh = 4, 32, 16
    Wb, Hb = W // N, Hh // N
    # interior footprint (quarter-block shift): not clipped, raw areas are the weights
    H = np.array([1.0, 0.0, 1.0, 0.0, 1.0, 1.0, 0.0, 0.0, 1.0])
    e, src, w, sw, clipped = oracle_mod.mix_weights(W, Hh, N, H, 3, 2, with_clipped=True)
    assert not e and not clipped
    assert w.tolist() == [0.5625, 0.1875, 0.1875, 0.0625] and sw == 1.0
    # last column: the H-neighbour falls outside -> clipped, sum of in-range areas 0.75
    e, src, w, sw, clipped = oracle_mod.mix_weights(W, Hh, N, H, Wb - 1, 2, with_clipped=True)
    assert not e and clipped and sw == 0.75
    # identity at the border: zero-weight neighbours outside do not count as clipping
    e, src, w, sw, clipped = oracle_mod.mix_weights(W, Hh, N, IDENT, Wb - 1, Hb - 1, with_clipped=True)
    assert not e and not clipped
    # through the step: last-column tilde = (0.5625 mu_s + 0.1875 mu_v) / 0.75 etc.
    st = np.zeros((6, Hb, Wb), np.float32)
    st[0] = np.arange(Wb * Hb, dtype=np.float32).reshape(Hb, Wb) * 3.0
    st[1] = 8.0
    st[2] = 12.0
    st[3:6] = st[0:3]
    A, _ = _probe_tilde_A(oracle_mod, st, H, N, W, Hh)
    mu_s, mu_v = st[0, 2, Wb - 1], st[0, 3, Wb - 1]
    expect_mu = (0.5625 / 0.75) * mu_s + (0.1875 / 0.75) * mu_v
    assert abs(A[0, 2, Wb - 1] - expect_mu) < 1e-4
    assert abs(A[2, 2, Wb - 1] - 12.0) < 1e-5
