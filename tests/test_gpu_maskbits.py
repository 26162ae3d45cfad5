"""Bit-packed masks (include/dmsgm.h DMSGM_MASK_BITS): the same classification (App. E
P:655-663, R14) stored as one bit per pixel, least significant bit first.  Checked bit
for bit against the oracle's byte masks packed by numpy.packbits, through every step API,
for both staged-kernel block sizes; unsupported configurations are refused."""
import numpy as np
import pytest

import synth
from gpu_util import params_pair, run_oracle

pytestmark = pytest.mark.gpu


def _pack(m):
    return np.packbits(m > 0, axis=-1, bitorder="little")


def _run(dm, frames, Hs, N, pg, mode):
    import torch
    T, S, H, W = frames.shape
    ctx = dm.Dmsgm(W, H, N, pg)
    ctx.set_mask_format(dm.DMSGM_MASK_BITS)
    mw = (W + 7) // 8
    mp = (mw + 15) // 16 * 16
    out = np.empty((T, S, H, mw), np.uint8)
    dev = torch.device("cuda", 0)
    if mode == "step_n":
        f = torch.from_numpy(frames).to(dev)
        m = torch.full((T, S, H, mp), 0xAB, dtype=torch.uint8, device=dev)
        ctx.step_n(T, f, torch.from_numpy(np.ascontiguousarray(Hs)).to(dev), m[..., :mw])
        torch.cuda.synchronize()
        out[:] = m[..., :mw].cpu().numpy()
        assert np.all(m[..., mw:].cpu().numpy() == 0xAB)              # nothing past the mask row
    elif mode == "host":
        hm = np.zeros((S, H, mp), np.uint8)
        for t in range(T):
            ctx.step_host(np.ascontiguousarray(frames[t]), np.ascontiguousarray(Hs[t]), hm[..., :mw])
            out[t] = hm[..., :mw]
    else:
        f = torch.empty((S, H, W), dtype=torch.uint8, device=dev)
        m = torch.zeros((S, H, mp), dtype=torch.uint8, device=dev)
        for t in range(T):
            f.copy_(torch.from_numpy(frames[t]))
            ctx.step(f, torch.from_numpy(np.ascontiguousarray(Hs[t])).to(dev), m[..., :mw])
            torch.cuda.synchronize()
            out[t] = m[..., :mw].cpu().numpy()
    state = np.stack([ctx.get_state(s) for s in range(S)])
    ctx.close()
    return out, state


@pytest.mark.parametrize("mode", ["step", "step_n", "host"])
def test_bits_c3_sequence(cuda_lib, oracle_mod, mode, monkeypatch):
    monkeypatch.delenv("DMSGM_KERNEL", raising=False)
    cfg = synth.config("C3", T=16)
    seq = synth.generate(cfg)
    pg, po = params_pair(cuda_lib, oracle_mod, cfg.S)
    gb, gs = _run(cuda_lib, seq.frames, seq.homographies, cfg.N, pg, mode)
    om, os_ = run_oracle(oracle_mod, seq.frames, seq.homographies, cfg.N, po, snapshot_every=cfg.T)
    for t in range(cfg.T):
        assert np.array_equal(gb[t], _pack(om[t])), f"{mode} frame {t}: bit masks differ"
    assert np.array_equal(gs.view(np.uint32), os_[cfg.T - 1].view(np.uint32))


@pytest.mark.parametrize("N,W,H,S", [(4, 256, 96, 3), (8, 512, 128, 2), (4, 1920, 64, 1)])
def test_bits_random_motion(cuda_lib, oracle_mod, N, W, H, S, monkeypatch):
    """Random near-identity homographies and textured frames, both block sizes."""
    monkeypatch.delenv("DMSGM_KERNEL", raising=False)
    rng = np.random.default_rng(W + N)
    T = 5
    yy, xx = np.mgrid[0:H, 0:W]
    base = 120 + 60 * np.sin(xx / 7.0) * np.cos(yy / 9.0)
    frames = np.clip(base[None, None] + rng.normal(0, 12, (T, S, H, W)), 0, 255).astype(np.uint8)
    Hs = np.stack([np.stack([synth.random_homography(rng, W, H, shift=1.0, rot_deg=0.05, zoom=0.001, persp=1e-7)
                             for _ in range(S)]) for _ in range(T)])
    pg, po = params_pair(cuda_lib, oracle_mod, S)
    gb, gs = _run(cuda_lib, frames, Hs, N, pg, "step")
    om, os_ = run_oracle(oracle_mod, frames, Hs, N, po, snapshot_every=T)
    for t in range(T):
        assert np.array_equal(gb[t], _pack(om[t])), f"frame {t}"
    assert np.array_equal(gs.view(np.uint32), os_[T - 1].view(np.uint32))


def test_bits_refused_where_unsupported(cuda_lib, oracle_mod, monkeypatch):
    monkeypatch.delenv("DMSGM_KERNEL", raising=False)
    pg, _ = params_pair(cuda_lib, oracle_mod, 1)
    for W, H, N in [(320, 64, 4), (128, 64, 1), (128, 64, 2), (512, 64, 16)]:   # Wb % 32 != 0, N not 4 / 8
        c = cuda_lib.Dmsgm(W, H, N, pg)
        with pytest.raises(cuda_lib.DmsgmError, match="EINVAL"):
            c.set_mask_format(cuda_lib.DMSGM_MASK_BITS)
        c.close()
    c = cuda_lib.Dmsgm(256, 64, 8, pg)
    c.set_band(0, 4, 1)
    with pytest.raises(cuda_lib.DmsgmError, match="EINVAL"):
        c.set_mask_format(cuda_lib.DMSGM_MASK_BITS)
    c.set_band(0, 8, 0)
    c.set_mask_format(cuda_lib.DMSGM_MASK_BITS)
    with pytest.raises(cuda_lib.DmsgmError, match="ESTATE"):
        c.set_band(0, 4, 1)
    c.set_mask_format(cuda_lib.DMSGM_MASK_BYTES)
    c.set_band(0, 4, 1)
    c.close()
