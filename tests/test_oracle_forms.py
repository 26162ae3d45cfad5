"""The kernel-order oracle (form 0) pinned against the plain definition (form 1).

Form 0 (oracle/dmsgm_oracle.c) evaluates the step in the canonical fp32 order that the
CUDA path reproduces bitwise: the displacement-form fp32 projection (R17), fused
multiply-add accumulation of the mix without dividing by sum W when the footprint is not
clipped (R6), a reciprocal then fma in Eqs. 3/5 (R10), and the fixed-sequence decay
exp (R18).  Form 1 (oracle/dmsgm_plain.c) is SURVEY.md §8(c)'s literal definition: fp64
projection, every mixed sum divided by sum W, IEEE division, libm exp in fp64.  Both
make the same decisions in exact arithmetic; their roundings differ.

Two comparisons over the paper-scale synthetic sequences (C1, C2 300 frames with and
without frequent decay, C3 300 frames, three C4 streams x 30 frames):

* per step ("teacher-forced"): from the SAME previous state (form 1's), one step of
  each form.  The tilde models after S1-S3 agree within the north_star tolerance
  (1e-4 relative / absolute for mu, var; 1e-5 for ages) on every live block; the new
  states agree within it on every block except those whose match or swap decision is a
  near-tie (relative margin < 1e-4 in form 1's own arithmetic) -- there the rounding
  order decides, and the two results are both correct readings of a tie; every
  differing mask pixel is either in such a block or within 1e-4 (relative) of its
  threshold.  The measured deviations are quoted in DESIGN.md §2 (R5/R6/R10/R17/R18).
* free-running: each form runs the whole sequence on its own; a near-tie decision
  makes the trajectories differ in that block from then on, so only the output
  masks are compared: they differ in < 0.01 % of all pixels.
"""
import math

import numpy as np
import pytest

import synth

TOL_MV = 1e-4      # north_star: fp32 means/variances within 1e-4 relative (absolute near 0)
TOL_AGE = 1e-5     # ages: the two forms round differently, so not bitwise; 1e-5 relative


def _params(oracle_mod, S, form, lam=0.001, theta_v=2500.0):
    return oracle_mod.OracleParams(theta_s=4.0, theta_d=4.0, var_init=255.0, age_cap=30.0, var_floor_match=0.1,
                                   var_floor_classify=0.25, decay_lambda=lam, decay_var_thresh=theta_v,
                                   num_streams=S, form=form)


EPS32 = 2.0 ** -24


def _close(a, b, tol, scale=None):
    """|a - b| <= tol * max(|b|, 1), plus 16 fp32 roundings of `scale` when given: the
    conditioning of Eq. 5's incremental form var~ + (V - var~)/(age~+1), whose result can
    be far smaller than var~ (a decayed, nearly zero age~ replaces var~ by V)."""
    a = a.astype(np.float64)
    b = b.astype(np.float64)
    lim = tol * np.maximum(np.abs(b), 1.0)
    if scale is not None:
        lim = lim + 16 * EPS32 * np.abs(scale.astype(np.float64))
    return np.abs(a - b) <= lim


def _near_ties(tilde, p, tie=1e-4):
    """Blocks whose S5 match or S7 swap decision lies within a relative `tie` of its
    threshold, evaluated in fp64 from form 1's tilde models (the decisions' inputs)."""
    t = tilde.astype(np.float64)
    muA, varA, ageA, muC, varC, ageC, M, live = t
    thA = p.theta_s * np.maximum(varA, p.var_floor_match)
    thC = p.theta_s * np.maximum(varC, p.var_floor_match)
    mA = np.abs((M - muA) ** 2 - thA) <= tie * thA
    mC = np.abs((M - muC) ** 2 - thC) <= tie * thC
    cap = p.age_cap
    # swap compares the post-S6 ages; the three branches give (A.age, C.age) =
    # (min(ageA+1, cap), ageC), (ageA, min(ageC+1, cap)), (ageA, 1)
    sw = np.zeros_like(mA)
    for a, c in ((np.minimum(ageA + 1, cap), ageC), (ageA, np.minimum(ageC + 1, cap)), (ageA, np.ones_like(ageA))):
        sw |= np.abs(c - a) <= tie * np.maximum(a, 1.0)
    return (mA | mC | sw) & (live > 0)


def _teacher_forced(oracle_mod, frames, Hs, N, lam=0.001, theta_v=2500.0):
    T, S, H, W = frames.shape
    Wb, Hb = W // N, H // N
    pk, pp = _params(oracle_mod, S, 0, lam, theta_v), _params(oracle_mod, S, 1, lam, theta_v)
    ok_o, pl_o = oracle_mod.Oracle(W, H, N, pk), oracle_mod.Oracle(W, H, N, pp)
    ok_o.set_tilde_probe(True)
    pl_o.set_tilde_probe(True)
    stats = dict(blocks=0, tie_blocks=0, diverged=0, mask_px=0, mask_diff=0, worst_mv=0.0, worst_age=0.0,
                 worst_tilde_mv=0.0, worst_tilde_age=0.0)
    prev = None
    for t in range(T):
        if prev is not None:
            for s in range(S):
                ok_o.set_state(s, prev[s])
        mk = ok_o.step(frames[t], Hs[t])
        mp = pl_o.step(frames[t], Hs[t])
        sk = np.stack([ok_o.get_state(s) for s in range(S)])
        sp = np.stack([pl_o.get_state(s) for s in range(S)])
        tk, tp = ok_o.tilde, pl_o.tilde
        # S1-S3: same exposure decisions, tilde models within tolerance on live blocks
        assert np.array_equal(tk[:, 7], tp[:, 7]), f"frame {t}: exposure differs"
        live = tp[:, 7] > 0
        for i, tol in ((0, TOL_MV), (1, TOL_MV), (3, TOL_MV), (4, TOL_MV), (2, TOL_AGE), (5, TOL_AGE)):
            good = _close(tk[:, i], tp[:, i], tol)
            assert good[live].all(), f"frame {t}: tilde plane {i} beyond tolerance on {(~good & live).sum()} blocks"
            d = (np.abs(tk[:, i].astype(np.float64) - tp[:, i]) / np.maximum(np.abs(tp[:, i]), 1.0))[live]
            key = "worst_tilde_age" if i in (2, 5) else "worst_tilde_mv"
            stats[key] = max(stats[key], float(d.max()) if d.size else 0.0)
        assert np.array_equal(tk[:, 6], tp[:, 6])                       # M: exact on both sides
        # S5-S9: new state within tolerance except at near-tie decisions
        ties = np.stack([_near_ties(tp[s], pp) for s in range(S)])
        good = np.ones((S, Hb, Wb), bool)
        for i, tol in ((0, TOL_MV), (1, TOL_MV), (3, TOL_MV), (4, TOL_MV), (2, TOL_AGE), (5, TOL_AGE)):
            scale = np.maximum(np.abs(tp[:, i]), np.abs(sp[:, i])) if i in (1, 4) else None
            good &= _close(sk[:, i], sp[:, i], tol, scale)
        bad = ~good
        assert not (bad & ~ties).any(), f"frame {t}: {(bad & ~ties).sum()} blocks differ without a near-tie"
        for i in range(6):
            scale = np.maximum(np.abs(sp[:, i]), 1.0)
            if i in (1, 4):
                scale = np.maximum(scale, np.abs(tp[:, i]))
            d = (np.abs(sk[:, i].astype(np.float64) - sp[:, i]) / scale)[good]
            key = "worst_age" if i in (2, 5) else "worst_mv"
            stats[key] = max(stats[key], float(d.max()) if d.size else 0.0)
        stats["blocks"] += good.size
        stats["tie_blocks"] += int(ties.sum())
        stats["diverged"] += int(bad.sum())
        # masks: a differing pixel lies in a near-tie block or within 1e-4 of its threshold
        diff = mk != mp
        if diff.any():
            s_i, y_i, x_i = np.nonzero(diff)
            tie_px = ties[s_i, y_i // N, x_i // N] | bad[s_i, y_i // N, x_i // N]
            I = frames[t][s_i, y_i, x_i].astype(np.float64)
            mu = sp[s_i, 0, y_i // N, x_i // N].astype(np.float64)
            T_ = pp.theta_d * np.maximum(sp[s_i, 1, y_i // N, x_i // N].astype(np.float64), pp.var_floor_classify)
            near = np.abs((I - mu) ** 2 - T_) <= 1e-4 * T_
            assert (tie_px | near).all(), f"frame {t}: mask pixels differ away from their threshold"
        stats["mask_diff"] += int(diff.sum())
        stats["mask_px"] += diff.size
        prev = sp
    ok_o.close()
    pl_o.close()
    assert stats["diverged"] <= 1e-5 * stats["blocks"], stats
    assert stats["mask_diff"] <= 1e-4 * stats["mask_px"], stats
    return stats


def _free_running(oracle_mod, frames, Hs, N, lam=0.001, theta_v=2500.0):
    T, S, H, W = frames.shape
    outs = []
    for form in (0, 1):
        o = oracle_mod.Oracle(W, H, N, _params(oracle_mod, S, form, lam, theta_v))
        outs.append(np.stack([o.step(frames[t], Hs[t]) for t in range(T)]))
        o.close()
    diff = int((outs[0] != outs[1]).sum())
    assert diff <= 1e-4 * outs[0].size, (diff, outs[0].size)
    return diff, outs[0].size


_SEQS = {}


def _seq(name, T=None, streams=None):
    key = (name, T, None if streams is None else tuple(streams))
    if key not in _SEQS:
        cfg = synth.config(name)
        s = synth.generate(cfg, T=T, streams=streams)
        _SEQS[key] = (cfg.N, s.frames, s.homographies)
    return _SEQS[key]


CASES = [
    ("C1", None, None, 0.001, 2500.0),
    ("C2", 300, None, 0.001, 2500.0),
    ("C2", 300, None, 0.01, 100.0),        # frequent decay: exercises R18 against libm exp
    ("C3", 300, None, 0.001, 2500.0),
    ("C4", 30, range(3), 0.001, 2500.0),
]


@pytest.mark.parametrize("name,T,streams,lam,theta_v", CASES,
                         ids=["C1", "C2x300", "C2x300-decay", "C3x300", "C4x3x30"])
def test_forms_per_step(oracle_mod, name, T, streams, lam, theta_v):
    N, fr, Hs = _seq(name, T, streams)
    st = _teacher_forced(oracle_mod, fr, Hs, N, lam, theta_v)
    print(name, st)


@pytest.mark.parametrize("name,T,streams,lam,theta_v", CASES,
                         ids=["C1", "C2x300", "C2x300-decay", "C3x300", "C4x3x30"])
def test_forms_free_running_masks(oracle_mod, name, T, streams, lam, theta_v):
    N, fr, Hs = _seq(name, T, streams)
    diff, n = _free_running(oracle_mod, fr, Hs, N, lam, theta_v)
    print(name, "mask pixels differing", diff, "of", n)


# --------------------------------------------------------------------------
# P14 against the plain form, and R18 against libm over its whole range
# --------------------------------------------------------------------------
def _ulps(a, b):
    return abs(int(np.float32(a).view(np.int32)) - int(np.float32(b).view(np.int32)))


def test_p14_decay_within_one_ulp_of_plain(oracle_mod):
    """P14: var~ = 3500, theta_v = 2500, lambda = 0.001, age~ = 10 -> 10 e^-1 (x = 1.0000000475,
    lambda being the fp32 0.001).  Form 0 within 1 ulp of form 1 and of the closed form."""
    N = 2
    st = np.zeros((6, 1, 1), np.float32)
    st[:, 0, 0] = [100.0, 3500.0, 10.0, 3.0, 1.0, 1.0]
    frame = np.full((N, N), 100, np.uint8)
    got = []
    for form in (0, 1):
        o = oracle_mod.Oracle(N, N, N, _params(oracle_mod, 1, form, 0.001, 2500.0))
        o.set_state(0, st)
        o.set_tilde_probe(True)
        o.step(frame[None], np.eye(3).reshape(1, 9))
        got.append(float(o.tilde[0, 2, 0, 0]))
        o.close()
    closed = np.float32(10.0) * np.float32(math.exp(-float(np.float32(0.001)) * 1000.0))
    assert got[1] == closed
    assert _ulps(got[0], got[1]) <= 1, got


def test_decay_factor_within_one_ulp_of_libm(oracle_mod):
    rng = np.random.default_rng(18)
    worst = 0
    for lam in (0.001, 0.01, 0.0003, 0.1, 1.0):
        lam32 = float(np.float32(lam))
        for d in np.float32(rng.uniform(0.0, 85.0 / lam32, 5000)):
            ref = np.float32(math.exp(-lam32 * float(d)))
            if ref < np.finfo(np.float32).tiny:
                continue
            worst = max(worst, _ulps(oracle_mod.decay_factor(lam32, float(d)), ref))
    assert worst <= 1, worst
    assert oracle_mod.decay_factor(0.001, 0.0) == 1.0
    assert oracle_mod.decay_factor(1.0, 86.0) == 0.0 and oracle_mod.decay_factor(1.0, 1e9) == 0.0
