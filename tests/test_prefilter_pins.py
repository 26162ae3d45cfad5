"""Pins of the preprocessing oracle (oracle/prefilter_oracle.c, readings R30-R34, SURVEY
§8(f) NEXT-2): checked against values the spec prints, closed forms, and independent
library routines (numpy float64 convolution, numpy median) -- never against a retyped
copy of the oracle's own loops.
"""
import os

import numpy as np
import pytest
import yaml

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "prefilter.yaml")


@pytest.fixture(scope="module")
def golden():
    with open(GOLDEN) as f:
        return yaml.safe_load(f)


def _exact_gauss(frame, taps64):
    """Separable Gaussian in float64 with edge clamping (numpy pad + correlate): the
    real-arithmetic result R31 rounds once."""
    k = len(taps64)
    h = (k - 1) // 2
    p = np.pad(frame.astype(np.float64), h, mode="edge")
    rows = np.zeros((p.shape[0], frame.shape[1]))
    for i in range(k):
        rows += taps64[i] * p[:, i:i + frame.shape[1]]
    out = np.zeros(frame.shape)
    for i in range(k):
        out += taps64[i] * rows[i:i + frame.shape[0], :]
    return out


def _taps64(size, sigma):
    c = (size - 1) / 2
    t = np.exp(-((np.arange(size) - c) ** 2) / (2 * sigma * sigma))
    return t / t.sum()


def test_taps_spec_values(oracle_mod, golden):
    for case in golden["taps"]:
        got = oracle_mod.gauss_taps(case["size"], case["sigma"])
        assert np.allclose(got, np.array(case["taps"], np.float32), rtol=0, atol=case["atol"]), (case, got)


@pytest.mark.parametrize("size,sigma", [(3, 1.0), (5, 1.0), (5, 0.7), (7, 2.0), (9, 1.5)])
def test_taps_closed_form(oracle_mod, size, sigma):
    t = oracle_mod.gauss_taps(size, sigma).astype(np.float64)
    c = (size - 1) // 2
    assert abs(t.sum() - 1.0) < 1e-6
    assert np.array_equal(t, t[::-1])                                     # symmetric about the centre
    for d in range(1, c + 1):                                             # Eq. 1 ratios
        assert t[c + d] / t[c] == pytest.approx(np.exp(-d * d / (2 * sigma * sigma)), rel=1e-6)
    with pytest.raises(ValueError):
        oracle_mod.gauss_taps(4, 1.0)


def test_constant_frame_identity(oracle_mod):
    for v in (0, 1, 42, 128, 254, 255):
        f = np.full((11, 13), v, np.uint8)
        assert np.all(oracle_mod.prefilter(f, 5, 1.0, 1) == v)
        assert np.all(oracle_mod.prefilter(f, 5, 1.0, 0) == v)


@pytest.mark.parametrize("size,sigma", [(3, 1.0), (5, 1.0), (7, 1.3)])
def test_gauss_matches_exact_convolution(oracle_mod, size, sigma):
    """fp32 separable pass vs the float64 separable convolution with edge clamping:
    the one rounding can differ only where the exact value is within fp32 error of a
    half-integer."""
    rng = np.random.default_rng(size)
    taps = oracle_mod.gauss_taps(size, sigma).astype(np.float64)     # the fp32 taps, exactly
    for shape in [(1, 1), (1, 17), (9, 1), (37, 53)]:
        f = rng.integers(0, 256, shape).astype(np.uint8)
        got = oracle_mod.prefilter(f, size, sigma, 0).astype(np.float64)
        exact = _exact_gauss(f, taps)
        ref = np.clip(np.rint(exact), 0, 255)
        diff = got != ref
        assert np.all(np.abs(got - exact) <= 0.5 + 1e-3)
        assert np.all(np.abs(exact[diff] - np.floor(exact[diff]) - 0.5) < 1e-3)


def test_impulse_response_is_outer_product(oracle_mod):
    f = np.zeros((15, 15), np.uint8)
    f[7, 7] = 255
    taps = _taps64(5, 1.0)
    got = oracle_mod.prefilter(f, 5, 1.0, 0).astype(np.float64)
    want = np.zeros((15, 15))
    want[5:10, 5:10] = 255 * np.outer(taps, taps)
    assert np.all(np.abs(got - np.rint(want)) <= 1)
    assert got[7, 7] == np.rint(255 * taps[2] * taps[2])


def test_median_spec_examples(oracle_mod, golden):
    for case in golden["median"]:
        f = np.array(case["frame"], np.uint8)
        got = oracle_mod.prefilter(f, 1, 1.0, case["radius"])
        for (y, x, v) in case["expect"]:
            assert got[y, x] == v, (case["id"], y, x, got)


@pytest.mark.parametrize("radius", [1, 2])
def test_median_matches_numpy(oracle_mod, radius):
    rng = np.random.default_rng(radius)
    for shape in [(1, 1), (2, 5), (23, 31)]:
        f = rng.integers(0, 256, shape).astype(np.uint8)
        p = np.pad(f, radius, mode="edge")
        k = 2 * radius + 1
        win = np.lib.stride_tricks.sliding_window_view(p, (k, k))
        want = np.median(win.reshape(*shape, k * k), axis=-1).astype(np.uint8)
        assert np.array_equal(oracle_mod.prefilter(f, 1, 1.0, radius), want)


def test_order_gauss_then_median(oracle_mod):
    """R34: the full filter is the median of the Gaussian output (and not the reverse)."""
    rng = np.random.default_rng(3)
    f = rng.integers(0, 256, (29, 41)).astype(np.uint8)
    both = oracle_mod.prefilter(f, 5, 1.0, 1)
    g = oracle_mod.prefilter(f, 5, 1.0, 0)
    assert np.array_equal(both, oracle_mod.prefilter(g, 1, 1.0, 1))
    m = oracle_mod.prefilter(f, 1, 1.0, 1)
    assert not np.array_equal(both, oracle_mod.prefilter(m, 5, 1.0, 0))


def test_prefilter_argument_errors(oracle_mod):
    f = np.zeros((4, 4), np.uint8)
    for bad in [(4, 1.0, 1), (5, 0.0, 1), (5, 1.0, -1), (5, 1.0, 5)]:
        with pytest.raises(ValueError):
            oracle_mod.prefilter(f, *bad)
