"""GPU parity of the frame-warp motion compensation (readings
R35-R37): the CUDA warp against the oracle's warp bit for bit, and whole steps in
DMSGM_MC_FRAME mode against the oracle run as "warp the frame, then step with H = I".
"""
import numpy as np
import pytest

import synth
from gpu_util import compare_masks, compare_state, params_pair, run_oracle

pytestmark = pytest.mark.gpu


def _homs(rng, S, W, H):
    out = np.empty((S, 9))
    for s in range(S):
        out[s] = synth.random_homography(rng, W, H, shift=rng.uniform(0, 6), rot_deg=1.0, zoom=0.02,
                                         persp=1e-4 / max(W, H))
    return out


@pytest.mark.parametrize("W,H,S", [(4, 1, 1), (8, 5, 2), (100, 37, 3), (256, 64, 2), (1920, 33, 1)])
def test_warp_bitwise(cuda_lib, oracle_mod, W, H, S):
    import torch
    rng = np.random.default_rng(W + H + S)
    yy, xx = np.mgrid[0:H, 0:W]
    frames = np.clip(120 + 80 * np.sin(xx / 6.0 + yy / 9.0) + rng.normal(0, 6, (S, H, W)), 0, 255).astype(np.uint8)
    Hs = _homs(rng, S, W, H)
    if S >= 2:
        Hs[1] = [1, 0, 0, 0, 1, 0, 0.01, 0, -0.5]       # w changes sign inside the frame: degenerate pixels
    dev = torch.device("cuda", 0)
    pitch = (W + 15) // 16 * 16
    fin = torch.zeros((S, H, pitch), dtype=torch.uint8, device=dev)
    fin[..., :W] = torch.from_numpy(frames).to(dev)
    fout = torch.full((S, H, pitch), 3, dtype=torch.uint8, device=dev)
    h = torch.from_numpy(Hs).to(dev)
    cuda_lib.warp_frames(fin[..., :W], h, fout[..., :W])
    torch.cuda.synchronize()
    got = fout[..., :W].cpu().numpy()
    assert np.all(fout[..., W:].cpu().numpy() == 3)                  # nothing written past the width
    want = oracle_mod.warp_frames(frames, Hs)
    assert np.array_equal(got, want), f"{(got != want).sum()} pixels differ"
    assert np.all(fout[..., W:].cpu().numpy() == 3)


def _run_frame_mode(dm, frames, Hs, N, params, mode, prefilter=None):
    import torch
    T, S, H, W = frames.shape
    ctx = dm.Dmsgm(W, H, N, params)
    ctx.set_motion(dm.DMSGM_MC_FRAME)
    if prefilter:
        ctx.set_prefilter(*prefilter)
    dev = torch.device("cuda", 0)
    pitch = (W + 15) // 16 * 16
    masks = np.empty_like(frames)
    h_all = torch.from_numpy(np.ascontiguousarray(Hs)).to(dev)
    if mode == "step_n":
        f = torch.zeros((T, S, H, pitch), dtype=torch.uint8, device=dev)
        f[..., :W] = torch.from_numpy(frames).to(dev)
        m = torch.zeros_like(f)
        ctx.step_n(T, f, h_all, m)
        torch.cuda.synchronize()
        masks[:] = m[..., :W].cpu().numpy()
    else:
        hf = np.zeros((S, H, pitch), np.uint8)
        hm = np.zeros((S, H, pitch), np.uint8)
        f = torch.zeros((S, H, pitch), dtype=torch.uint8, device=dev)
        m = torch.zeros_like(f)
        for t in range(T):
            if mode == "host":
                hf[..., :W] = frames[t]
                ctx.step_host(hf, np.ascontiguousarray(Hs[t]), hm)
                masks[t] = hm[..., :W]
            else:
                f[..., :W] = torch.from_numpy(frames[t]).to(dev)
                ctx.step(f, h_all[t], m)
                torch.cuda.synchronize()
                masks[t] = m[..., :W].cpu().numpy()
    state = np.stack([ctx.get_state(s) for s in range(S)])
    ctx.close()
    return masks, state


@pytest.mark.parametrize("mode", ["step", "step_n", "host"])
@pytest.mark.parametrize("prefilter", [None, (5, 1.0, 1)])
def test_step_frame_mode(cuda_lib, oracle_mod, mode, prefilter):
    cfg = synth.config("C2", T=10, S=2)
    seq = synth.generate(cfg)
    pg, po = params_pair(cuda_lib, oracle_mod, cfg.S)
    gm, gs = _run_frame_mode(cuda_lib, seq.frames, seq.homographies, cfg.N, pg, mode, prefilter)
    frames = seq.frames if not prefilter else oracle_mod.prefilter_frames(seq.frames, *prefilter)
    warped = oracle_mod.warp_frames(frames, seq.homographies)                  # R35: warp, then H = I
    ident = np.broadcast_to(np.eye(3).reshape(9), seq.homographies.shape).copy()
    om, os_ = run_oracle(oracle_mod, warped, ident, cfg.N, po, snapshot_every=1)
    compare_state(gs, os_[cfg.T - 1], where=mode)
    for t in range(cfg.T):
        compare_masks(gm[t], om[t], warped[t], (os_[t][:, 0], os_[t][:, 1]), cfg.N, where=f"{mode} t={t}")


def test_motion_mode_errors(cuda_lib, oracle_mod):
    import torch
    pg, _ = params_pair(cuda_lib, oracle_mod, 1)
    c = cuda_lib.Dmsgm(64, 64, 8, pg)
    with pytest.raises(cuda_lib.DmsgmError):
        c.set_motion(2)
    c.set_motion(cuda_lib.DMSGM_MC_FRAME)
    assert c.info.kernels_per_step == 2
    with pytest.raises(cuda_lib.DmsgmError, match="ESTATE"):
        c.set_band(0, 4, 1)
    c.set_motion(cuda_lib.DMSGM_MC_MODELS)
    assert c.info.kernels_per_step == 1
    c.close()
    x = torch.zeros((1, 8, 6), dtype=torch.uint8, device="cuda")                # width % 4 != 0
    with pytest.raises(cuda_lib.DmsgmError):
        cuda_lib.warp_frames(x, torch.zeros((1, 9), dtype=torch.float64, device="cuda"), x)


def _translation(dx, dy):
    return np.array([1, 0, dx, 0, 1, dy, 0, 0, 1], dtype=np.float64)


def _similarity(W, H, zoom, rot_deg, dx=0.0, dy=0.0):
    cx, cy = W / 2.0, H / 2.0
    th = rot_deg * np.pi / 180.0
    c, s = zoom * np.cos(th), zoom * np.sin(th)
    A = np.array([[c, -s, cx + dx - c * cx + s * cy], [s, c, cy + dy - s * cx - c * cy], [0, 0, 1.0]])
    return A.reshape(9)


@pytest.mark.parametrize("case", ["shifts", "half_pixel", "far_out", "zoom_rot", "fallback", "unaligned_pitch"])
def test_warp_fast_tiles(cuda_lib, oracle_mod, case):
    """The fast-tile path (border-replicated box at a fixed pitch, magic-number floor and
    byte conversion, paired arithmetic) and the fallbacks it hands over to, bit for bit
    against the oracle: border tiles with samples far outside the frame, exact integer
    and half-pixel positions (fx = 0, rounding ties), zoom/rotation/perspective at 1080p
    width, maps whose source box exceeds the fixed pitch or row budget (clamped staged
    box / global gathers), and a row pitch that is not a multiple of 16 (no fast tiles)."""
    import torch
    rng = np.random.default_rng(sum(map(ord, case)))
    W, H = (1920, 72) if case in ("zoom_rot", "fallback") else (512, 80)
    homs = {
        "shifts": [_translation(3, -2), _translation(-7.25, 5.5), _translation(1.0 / 3, -40.7), _translation(37, 0.125)],
        "half_pixel": [_translation(0.5, 0), _translation(-0.5, 0.5), _translation(2.5, -1.5), _translation(0, 0)],
        "far_out": [_translation(-300, 3), _translation(5, 200), _translation(600, -600), _translation(-1.5, -70)],
        "zoom_rot": [_similarity(W, H, 1.0005, 0.05, 1.3, -0.7), _similarity(W, H, 0.98, -2.0, -3, 2),
                     synth.random_homography(rng, W, H, shift=4, rot_deg=3, zoom=0.05, persp=2e-5),
                     _similarity(W, H, 1.2, 0.0)],
        "fallback": [_similarity(W, H, 3.0, 0.0), _similarity(W, H, 1.0, 30.0), _similarity(W, H, 0.3, 5.0, 9, 9),
                     np.array([1, 0, 0, 0, 1, 0, 2e-3, 0, 1.0])],
        "unaligned_pitch": [_translation(3, -2), _similarity(W, H, 1.01, 1.0, 2, 2), _translation(-0.5, 20),
                            _translation(0, 0)],
    }[case]
    Hs = np.stack(homs)
    S = len(Hs)
    yy, xx = np.mgrid[0:H, 0:W]
    frames = np.clip(120 + 90 * np.sin(xx / 5.0 + yy / 7.0) + rng.normal(0, 20, (S, H, W)), 0, 255).astype(np.uint8)
    dev = torch.device("cuda", 0)
    pitch = W + 4 if case == "unaligned_pitch" else W
    fin = torch.zeros((S, H, pitch), dtype=torch.uint8, device=dev)
    fin[..., :W] = torch.from_numpy(frames).to(dev)
    fout = torch.full((S, H, pitch), 7, dtype=torch.uint8, device=dev)
    cuda_lib.warp_frames(fin[..., :W], torch.from_numpy(Hs).to(dev), fout[..., :W])
    torch.cuda.synchronize()
    got = fout[..., :W].cpu().numpy()
    assert np.all(fout[..., W:].cpu().numpy() == 7)                  # nothing written past the width
    want = oracle_mod.warp_frames(frames, Hs)
    for s in range(S):
        assert np.array_equal(got[s], want[s]), f"{case} stream {s}: {(got[s] != want[s]).sum()} pixels differ"
