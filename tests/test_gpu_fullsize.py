"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

C4: 32 streams of 1920x1080, N=4; C5: 64 streams of 3840x2160, N=8.  The GPU runs the
whole batch (same grid as the bench); the oracle recomputes a sample of streams in full
(streams are independent, so a stream's result does not depend on the rest of the batch;
test_batch_invariance pins that).  Non-sampled streams carry copies of sampled content.
"""
import numpy as np
import pytest

import synth
from gpu_util import compare_masks, compare_state, params_pair

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.mark.parametrize("name,T,sample", [("C4", 3, [0, 17, 31]), ("C5", 2, [5, 63])])
def test_fullsize_sampled_streams(cuda_lib, oracle_mod, name, T, sample, monkeypatch):
    monkeypatch.delenv("DMSGM_KERNEL", raising=False)       # the bench's kernel
    import torch
    dm = cuda_lib
    cfg = synth.config(name, T=T)
    seq = synth.generate(cfg, streams=sample)
    S, H, W, N = cfg.S, cfg.H, cfg.W, cfg.N
    src = [sample.index(s) if s in sample else s % len(sample) for s in range(S)]
    pg, po = params_pair(dm, oracle_mod, S)
    ctx = dm.Dmsgm(W, H, N, pg)
    f = torch.empty((S, H, W), dtype=torch.uint8, device="cuda")
    m = torch.empty_like(f)
    o_params = params_pair(dm, oracle_mod, len(sample))[1]
    o = oracle_mod.Oracle(W, H, N, o_params)
    for t in range(T):
        f.copy_(torch.from_numpy(seq.frames[t][src]))
        h = torch.from_numpy(np.ascontiguousarray(seq.homographies[t][src])).cuda()
        ctx.step(f, h, m)
        om = o.step(seq.frames[t], seq.homographies[t])
        torch.cuda.synchronize()
        gm = m.cpu().numpy()
        ost = np.stack([o.get_state(j) for j in range(len(sample))])
        gst = np.stack([ctx.get_state(s) for s in sample])
        compare_state(gst, ost, where=f"{name} t={t}")
        compare_masks(gm[sample], om, seq.frames[t], (ost[:, 0], ost[:, 1]), N, where=f"{name} t={t}")
    ctx.close()
    o.close()


def test_fullsize_c5b_bands(cuda_lib, oracle_mod, monkeypatch):
    """C5b: one 4K stream split into 8 row bands (34 x 6 + 33 x 2 block rows) on concurrent
    CUDA streams, through per-band CUDA graphs -- the bench's configuration -- equals the
    whole-frame oracle on every frame."""
    monkeypatch.delenv("DMSGM_KERNEL", raising=False)
    import torch

    from paper_1702_05156_b200.band import BandGroup, band_rows, halo_for
    dm = cuda_lib
    cfg = synth.config("C5b", T=3)
    seq = synth.generate(cfg)
    W, H, N, G, T = cfg.W, cfg.H, cfg.N, 8, cfg.T
    bands = band_rows(H // N, G)
    halo = halo_for(W, H, N, seq.homographies.reshape(-1, 9), bands)
    pg, po = params_pair(dm, oracle_mod, 1)
    dev = torch.device("cuda", 0)
    streams = [torch.cuda.Stream(dev) for _ in range(G)]
    grp = BandGroup(W, H, N, pg, G, halo, streams=streams)
    fb = [torch.from_numpy(np.ascontiguousarray(seq.frames[:, :, b.row0 * N:b.row1 * N])).to(dev) for b in bands]
    mb = [torch.zeros_like(f) for f in fb]
    h = torch.from_numpy(np.ascontiguousarray(seq.homographies)).to(dev)
    torch.cuda.synchronize()
    grp.step_n(T, fb, h, mb)
    torch.cuda.synchronize()
    assert grp.status() == [0] * G
    gm = np.concatenate([m.cpu().numpy() for m in mb], axis=2)          # [T][1][H][W]
    gst = grp.get_state(0)
    grp.close()
    om, ost = oracle_mod.Oracle(W, H, N, po), None
    for t in range(T):
        o_mask = om.step(seq.frames[t], seq.homographies[t])
        ost = np.stack([om.get_state(0)])
        compare_masks(gm[t], o_mask, seq.frames[t], (ost[:, 0], ost[:, 1]), N, where=f"C5b t={t}")
    compare_state(gst[None], ost, where="C5b final")
    om.close()
