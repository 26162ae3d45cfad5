"""Pins of the frame-warp oracle (oracle/warp_oracle.c, readings R35-R37, SURVEY §8(f)
NEXT-3: App. F's warpPerspective(..., INTER_LINEAR | WARP_INVERSE_MAP)) against closed
forms and an independent library routine (scipy.ndimage.map_coordinates, order 1,
edge mode) -- never against a retyped copy of the oracle's loop.
"""
import numpy as np
import pytest


def _ramp(h, w):
    y, x = np.mgrid[0:h, 0:w]
    return np.clip(3 * x + 2 * y + 10, 0, 255).astype(np.uint8)


def test_identity_is_exact(oracle_mod):
    rng = np.random.default_rng(1)
    f = rng.integers(0, 256, (17, 23)).astype(np.uint8)
    assert np.array_equal(oracle_mod.warp_frame(f, np.eye(3)), f)
    assert np.array_equal(oracle_mod.warp_frame(f, 2.5 * np.eye(3)), f)        # projective scale cancels


@pytest.mark.parametrize("tx,ty", [(1, 0), (0, -2), (3, 5), (-4, 1)])
def test_integer_translation_is_index_shift(oracle_mod, tx, ty):
    """H_t maps frame t to frame t-1 by (+tx, +ty) (R3): out(x, y) = frame(x - tx, y - ty),
    border pixels repeated (R37)."""
    rng = np.random.default_rng(abs(tx * 10 + ty))
    f = rng.integers(0, 256, (12, 15)).astype(np.uint8)
    H = np.array([[1, 0, tx], [0, 1, ty], [0, 0, 1]], np.float64)
    y, x = np.mgrid[0:12, 0:15]
    want = f[np.clip(y - ty, 0, 11), np.clip(x - tx, 0, 14)]
    assert np.array_equal(oracle_mod.warp_frame(f, H), want)


def test_half_pixel_translation_averages(oracle_mod):
    f = _ramp(6, 20)
    f[:, ::3] += 1                                             # odd sums: exercise ties to even
    H = np.array([[1, 0, 0.5], [0, 1, 0], [0, 0, 1]], np.float64)
    got = oracle_mod.warp_frame(f, H).astype(np.int64)
    xm = np.clip(np.arange(20) - 1, 0, 19)
    want = np.rint((f[:, xm].astype(np.float64) + f.astype(np.float64)) / 2)
    assert np.array_equal(got, want)


def test_matches_scipy_bilinear(oracle_mod):
    from scipy.ndimage import map_coordinates
    rng = np.random.default_rng(7)
    h, w = 40, 56
    y, x = np.mgrid[0:h, 0:w].astype(np.float64)
    f = np.clip(128 + 90 * np.sin(x / 5.0) * np.cos(y / 7.0), 0, 255).astype(np.uint8)
    for _ in range(8):
        H = np.eye(3) + rng.normal(0, 1, (3, 3)) * np.array([[2e-3, 2e-3, 1.5], [2e-3, 2e-3, 1.5], [2e-5, 2e-5, 0]])
        Hi = np.linalg.inv(H)
        X, Y = x + 0.5, y + 0.5
        wn = Hi[2, 0] * X + Hi[2, 1] * Y + Hi[2, 2]
        sx = (Hi[0, 0] * X + Hi[0, 1] * Y + Hi[0, 2]) / wn - 0.5
        sy = (Hi[1, 0] * X + Hi[1, 1] * Y + Hi[1, 2]) / wn - 0.5
        ref = map_coordinates(f.astype(np.float64), [sy, sx], order=1, mode="nearest")
        got = oracle_mod.warp_frame(f, H).astype(np.float64)
        d = np.abs(got - ref)
        assert d.max() <= 0.5 + 2e-3, d.max()                # one rounding of the same interpolant
        assert np.mean(got == np.rint(ref)) > 0.995


def test_warp_then_inverse_smooth(oracle_mod):
    """warp then inverse-warp of a smooth image stays within 2 levels inside."""
    h, w = 48, 64
    y, x = np.mgrid[0:h, 0:w].astype(np.float64)
    f = np.clip(120 + 60 * np.sin(x / 9.0 + y / 13.0), 0, 255).astype(np.uint8)
    H = np.array([[1.001, 0.002, 1.3], [-0.001, 0.999, -0.7], [1e-6, 0, 1]])
    back = oracle_mod.warp_frame(oracle_mod.warp_frame(f, H), np.linalg.inv(H))
    inner = (slice(4, h - 4), slice(4, w - 4))
    assert np.abs(back[inner].astype(int) - f[inner].astype(int)).max() <= 2


def test_degenerate_maps_leave_pixels(oracle_mod):
    rng = np.random.default_rng(3)
    f = rng.integers(0, 256, (9, 11)).astype(np.uint8)
    for H in (np.zeros((3, 3)),                                        # singular: no inverse
              np.array([[1, 0, 1e9], [0, 1, 0], [0, 0, 1.0]])):        # 2^20 px or more
        assert np.array_equal(oracle_mod.warp_frame(f, H), f)
    # inverse map with w = 1 - X/2: non-positive for every pixel centre X >= 2.5 (x >= 2)
    H = np.linalg.inv(np.array([[1, 0, 0], [0, 1, 0], [-0.5, 0, 1.0]]))
    assert np.array_equal(oracle_mod.warp_frame(f, H)[:, 2:], f[:, 2:])
