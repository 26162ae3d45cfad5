"""GPU parity of the preprocessing (readings R30-R34): the CUDA
filter kernel against the oracle's filter, bit for bit, and the whole step with the
filter on against the oracle run on the oracle-filtered frames.
"""
import numpy as np
import pytest

import synth
from gpu_util import compare_masks, compare_state, params_pair, run_oracle

pytestmark = pytest.mark.gpu

COMBOS = [(1, 1.0, 0), (1, 1.0, 1), (3, 1.0, 0), (3, 0.8, 1), (5, 1.0, 0), (5, 1.0, 1), (7, 1.5, 1), (7, 2.0, 0)]


@pytest.mark.parametrize("gs,sigma,mr", COMBOS)
# sizes: single pixel rows, ragged 240-column strips and 120-row bands of the streaming
# kernel (244 = 240 + 4, 484 = 2 x 240 + 4, 248 = 240 + 8, 121 = 120 + 1, 241 = 2 x 120 + 1),
# a 1080p-wide frame of 2 rows
@pytest.mark.parametrize("W,H,S", [(4, 1, 1), (8, 3, 2), (12, 2, 1), (100, 45, 2), (256, 64, 1), (132, 33, 3),
                                   (244, 81, 1), (1920, 2, 1), (364, 121, 2), (484, 241, 1), (248, 120, 2)])
def test_filter_bitwise(cuda_lib, oracle_mod, gs, sigma, mr, W, H, S):
    import torch
    rng = np.random.default_rng(W * 1000 + H + gs + mr)
    frames = rng.integers(0, 256, (S, H, W)).astype(np.uint8)
    if W >= 64:      # smooth content plus noise, as in the bench's sequences
        yy, xx = np.mgrid[0:H, 0:W]
        frames = np.clip(120 + 60 * np.sin(xx / 7.0 + yy / 11.0) + rng.normal(0, 8, (S, H, W)), 0, 255).astype(np.uint8)
    dev = torch.device("cuda", 0)
    pitch = (W + 15) // 16 * 16
    fin = torch.zeros((S, H, pitch), dtype=torch.uint8, device=dev)
    fin[..., :W] = torch.from_numpy(frames).to(dev)
    fout = torch.full((S, H, pitch), 7, dtype=torch.uint8, device=dev)
    cuda_lib.prefilter(fin[..., :W], fout[..., :W], gs, sigma, mr)
    torch.cuda.synchronize()
    got = fout[..., :W].cpu().numpy()
    want = oracle_mod.prefilter_frames(frames, gs, sigma, mr)
    assert np.array_equal(got, want), f"{(got != want).sum()} pixels differ"
    assert np.all(fout[..., W:].cpu().numpy() == 7)                  # nothing written past the width


def test_filter_argument_errors(cuda_lib):
    import torch
    x = torch.zeros((1, 8, 16), dtype=torch.uint8, device="cuda")
    for bad in [(4, 1.0, 1), (9, 1.0, 0), (5, 0.0, 1), (5, 1.0, 2)]:
        with pytest.raises(cuda_lib.DmsgmError):
            cuda_lib.prefilter(x, x, *bad)
    y = torch.zeros((1, 8, 18), dtype=torch.uint8, device="cuda")[..., :16]   # row pitch 18: not 4-byte aligned
    with pytest.raises(cuda_lib.DmsgmError):
        cuda_lib.prefilter(y, x, 5, 1.0, 1)


def _run_step_with_prefilter(dm, frames, Hs, N, params, mode):
    import torch
    T, S, H, W = frames.shape
    ctx = dm.Dmsgm(W, H, N, params)
    ctx.set_prefilter(5, 1.0, 1)
    assert ctx.info.kernels_per_step == 2
    dev = torch.device("cuda", 0)
    pitch = (W + 15) // 16 * 16
    masks = np.empty_like(frames)
    if mode == "step_n":
        f = torch.zeros((T, S, H, pitch), dtype=torch.uint8, device=dev)
        f[..., :W] = torch.from_numpy(frames).to(dev)
        m = torch.zeros_like(f)
        ctx.step_n(T, f, torch.from_numpy(np.ascontiguousarray(Hs)).to(dev), m)
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
                ctx.step(f, torch.from_numpy(np.ascontiguousarray(Hs[t])).to(dev), m)
                torch.cuda.synchronize()
                masks[t] = m[..., :W].cpu().numpy()
    state = np.stack([ctx.get_state(s) for s in range(S)])
    ctx.close()
    return masks, state


@pytest.mark.parametrize("mode", ["step", "step_n", "host"])
def test_step_with_prefilter(cuda_lib, oracle_mod, mode):
    cfg = synth.config("C2", T=12, S=2)
    seq = synth.generate(cfg)
    pg, po = params_pair(cuda_lib, oracle_mod, cfg.S)
    gm, gs = _run_step_with_prefilter(cuda_lib, seq.frames, seq.homographies, cfg.N, pg, mode)
    filtered = oracle_mod.prefilter_frames(seq.frames, 5, 1.0, 1)            # R34: filter, then the step
    om, os_ = run_oracle(oracle_mod, filtered, seq.homographies, cfg.N, po, snapshot_every=1)
    compare_state(gs, os_[cfg.T - 1], where=mode)
    for t in range(cfg.T):
        compare_masks(gm[t], om[t], filtered[t], (os_[t][:, 0], os_[t][:, 1]), cfg.N, where=f"{mode} t={t}")


def test_prefilter_band_mode_refused(cuda_lib, oracle_mod):
    pg, _ = params_pair(cuda_lib, oracle_mod, 1)
    c = cuda_lib.Dmsgm(64, 64, 8, pg)
    c.set_band(0, 4, 1)
    with pytest.raises(cuda_lib.DmsgmError, match="ESTATE"):
        c.set_prefilter(5, 1.0, 1)
    c.set_band(0, 8, 0)
    c.set_prefilter(5, 1.0, 1)
    with pytest.raises(cuda_lib.DmsgmError, match="ESTATE"):
        c.set_band(0, 4, 1)
    c.set_prefilter(1, 1.0, 0)                                                # off again
    assert c.info.kernels_per_step == 1
    c.close()
