"""Helpers for the -m gpu parity tests: run the CUDA path and the oracle on the same inputs."""
from __future__ import annotations

import numpy as np

# north_star tolerances (BASELINE.json): fp32 means/variances within 1e-4 relative,
# ages exactly, masks differing in <= 0.01 % of pixels, each within 1e-4 of its threshold.
REL_TOL = 1e-4
MASK_FRAC = 1e-4
THRESH_TOL = 1e-4


def params_pair(dm, oracle_mod, S, **kw):
    base = dict(theta_s=4.0, theta_d=4.0, var_init=255.0, age_cap=30.0, var_floor_match=0.1,
                var_floor_classify=0.25, decay_lambda=0.001, decay_var_thresh=2500.0,
                num_streams=S, update_rule=0, classify_rule=0)
    base.update(kw)
    return dm.Params(**base), oracle_mod.OracleParams(**base)


def run_gpu(dm, frames, Hs, N, params, init_states=None, mode="step", snapshot_every=1):
    """frames u8 [T][S][H][W], Hs f64 [T][S][9] -> (masks [T][S][H][W], states {t: [S][6][Hb][Wb]})."""
    import torch
    T, S, H, W = frames.shape
    ctx = dm.Dmsgm(W, H, N, params)
    if init_states is not None:
        for s in range(S):
            ctx.set_state(s, init_states[s])
    dev = torch.device("cuda", 0)
    pitch = (W + 15) // 16 * 16
    masks = np.empty_like(frames)
    states = {}
    if mode == "step_n":
        f = torch.zeros((T, S, H, pitch), dtype=torch.uint8, device=dev)
        f[..., :W] = torch.from_numpy(frames).to(dev)
        h = torch.from_numpy(np.ascontiguousarray(Hs)).to(dev)
        m = torch.zeros((T, S, H, pitch), dtype=torch.uint8, device=dev)
        ctx.step_n(T, f, h, m)
        torch.cuda.synchronize()
        masks[:] = m[..., :W].cpu().numpy()
        states[T - 1] = np.stack([ctx.get_state(s) for s in range(S)])
    else:
        f = torch.zeros((S, H, pitch), dtype=torch.uint8, device=dev)
        m = torch.zeros((S, H, pitch), dtype=torch.uint8, device=dev)
        hf = np.zeros((S, H, pitch), np.uint8)
        hm = np.zeros((S, H, pitch), np.uint8)
        for t in range(T):
            if mode == "host":
                hf[..., :W] = frames[t]
                ctx.step_host(hf, np.ascontiguousarray(Hs[t]), hm)
                masks[t] = hm[..., :W]
            else:
                f[..., :W] = torch.from_numpy(frames[t]).to(dev)
                h = torch.from_numpy(np.ascontiguousarray(Hs[t])).to(dev)
                ctx.step(f, h, m)
                torch.cuda.synchronize()
                masks[t] = m[..., :W].cpu().numpy()
            if (t % snapshot_every == 0) or t == T - 1:
                states[t] = np.stack([ctx.get_state(s) for s in range(S)])
    ctx.close()
    return masks, states


def run_oracle(oracle_mod, frames, Hs, N, params, init_states=None, snapshot_every=1):
    T, S, H, W = frames.shape
    o = oracle_mod.Oracle(W, H, N, params)
    if init_states is not None:
        for s in range(S):
            o.set_state(s, init_states[s])
    masks = np.empty_like(frames)
    states = {}
    for t in range(T):
        masks[t] = o.step(frames[t], Hs[t])
        if (t % snapshot_every == 0) or t == T - 1:
            states[t] = np.stack([o.get_state(s) for s in range(S)])
    o.close()
    return masks, states


def compare_state(got, ref, where=""):
    """north_star tolerance on models; returns the number of bitwise-different values."""
    assert got.shape == ref.shape, (got.shape, ref.shape)
    for m in (0, 3):
        for p, name in ((0, "mu"), (1, "var")):
            g, r = got[:, m + p], ref[:, m + p]
            err = np.abs(g.astype(np.float64) - r.astype(np.float64))
            lim = REL_TOL * np.maximum(np.abs(r.astype(np.float64)), 1.0)
            bad = err > lim
            assert not bad.any(), f"{where} {name}{'AC'[m // 3]}: {bad.sum()} values off, max err {err.max()}"
        ga, ra = got[:, m + 2], ref[:, m + 2]
        assert np.array_equal(ga, ra), f"{where} age{'AC'[m // 3]}: {(ga != ra).sum()} ages differ"
    return int((got.view(np.uint32) != ref.view(np.uint32)).sum())


def compare_masks(got, ref, frames, ref_state_mu_var, N, theta_d=4.0, f_c=0.25, where=""):
    """north_star mask bar: <= 0.01 % differing pixels, each within 1e-4 of its threshold."""
    diff = got != ref
    n = int(diff.sum())
    if n == 0:
        return 0
    assert n <= MASK_FRAC * got.size, f"{where}: {n} mask pixels differ ({n / got.size:.2e})"
    mu, var = ref_state_mu_var
    idx = np.argwhere(diff)
    for (s, y, x) in idx:
        I = float(frames[s, y, x])
        m = float(mu[s, y // N, x // N])
        T = theta_d * max(float(var[s, y // N, x // N]), f_c)
        assert abs((I - m) ** 2 - T) <= THRESH_TOL * max(T, 1.0), f"{where}: pixel {(s, y, x)} far from threshold"
    return n
