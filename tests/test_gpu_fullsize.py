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


@pytest.mark.parametrize("name,replays,sample", [("C4", 3, [0, 13, 31]), ("C5", 1, [7, 62])])
def test_fullsize_bench_bytes(cuda_lib, oracle_mod, name, replays, sample, monkeypatch):
    """The bench's own inputs in the bench's launch path: the ring rendered on the GPU by
    synth.generate_device (torch backend -- its bytes differ from the numpy parity inputs,
    so they must pass through the oracle too), repeated to bench.GRAPH_T slots, warmed up
    by single dmsgm_step launches and then stepped by dmsgm_step_n CUDA-graph replays with
    programmatic dependent launch and early frame loads -- C4: 3 replays (123 steps), C5:
    1 replay (43 steps).  The frames are copied to the host; sampled streams are recomputed
    by the oracle over the same slot sequence; every mask of the sampled streams and the
    state at the end of every replay must equal the oracle's bitwise."""
    monkeypatch.delenv("DMSGM_KERNEL", raising=False)
    import torch

    import bench
    dm = cuda_lib
    cfg = synth.config(name + "ring")
    S, H, W, N = cfg.S, cfg.H, cfg.W, cfg.N
    ring, Hs = synth.generate_device(cfg, T=bench.RING, device="cuda:0")
    GT = bench.GRAPH_T
    frames = ring.repeat(GT // bench.RING, 1, 1, 1)
    del ring
    Hs_all = np.ascontiguousarray(np.tile(Hs, (GT // bench.RING, 1, 1)))
    hdev = torch.from_numpy(Hs_all).cuda()
    masks = torch.zeros_like(frames)
    host_frames = frames[:, sample].cpu().numpy()          # [GT][len(sample)][H][W]
    pg, po = params_pair(dm, oracle_mod, S)
    ctx = dm.Dmsgm(W, H, N, pg)
    o = oracle_mod.Oracle(W, H, N, params_pair(dm, oracle_mod, len(sample))[1])
    warm = [0, 1, 2]
    for i in warm:                                         # the bench's warm-up single steps
        ctx.step(frames[i], hdev[i], masks[i])
        o.step(host_frames[i], Hs_all[i][sample])
    ctx.step_n(GT, frames, hdev, masks)                    # capture + first replay
    for r in range(replays):
        if r:
            ctx.step_n(GT, frames, hdev, masks)
        torch.cuda.synchronize()
        gm = masks[:, sample].cpu().numpy()
        for t in range(GT):
            om = o.step(host_frames[t], Hs_all[t][sample])
            assert np.array_equal(gm[t], om), f"{name} replay {r} step {t}: {(gm[t] != om).sum()} pixels differ"
        gst = np.stack([ctx.get_state(s) for s in sample])
        ost = np.stack([o.get_state(j) for j in range(len(sample))])
        compare_state(gst, ost, where=f"{name} replay {r}")
        assert np.array_equal(gst.view(np.uint32), ost.view(np.uint32)), f"{name} replay {r}: states differ"
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


@pytest.mark.parametrize("W,H,N,S,T", [(7680, 4320, 4, 1, 2), (64, 48, 4, 700, 3), (3840, 2160, 1, 1, 2)])
def test_extreme_sizes(cuda_lib, oracle_mod, W, H, N, S, T, monkeypatch):
    """8K frames (2 M blocks per stream), 700 tiny streams (many more work items than
    resident CTAs: the dynamic item counter wraps many times), and a per-pixel 4K frame
    (8.3 M models) against the oracle -- bitwise on masks and states."""
    monkeypatch.delenv("DMSGM_KERNEL", raising=False)
    import torch
    from gpu_util import run_oracle
    rng = np.random.default_rng(W + S)
    yy, xx = np.mgrid[0:H, 0:W]
    base = (120 + 60 * np.sin(xx / 13.0) * np.cos(yy / 17.0)).astype(np.float64)
    frames = np.clip(base[None, None] + rng.normal(0, 3, (T, S, H, W)), 0, 255).astype(np.uint8)
    Hs = np.empty((T, S, 9))
    for t in range(T):
        for s in range(S):
            Hs[t, s] = synth.random_homography(rng, W, H, shift=1.5, rot_deg=0.05, zoom=0.001, persp=1e-7)
    pg, po = params_pair(cuda_lib, oracle_mod, S)
    ctx = cuda_lib.Dmsgm(W, H, N, pg)
    f = torch.empty((S, H, W), dtype=torch.uint8, device="cuda")
    m = torch.empty_like(f)
    gm = np.empty_like(frames)
    for t in range(T):
        f.copy_(torch.from_numpy(frames[t]))
        ctx.step(f, torch.from_numpy(np.ascontiguousarray(Hs[t])).cuda(), m)
        torch.cuda.synchronize()
        gm[t] = m.cpu().numpy()
    gst = np.stack([ctx.get_state(s) for s in range(S)])
    ctx.close()
    om, os_ = run_oracle(oracle_mod, frames, Hs, N, po, snapshot_every=T)
    compare_state(gst, os_[T - 1], where=f"{W}x{H} N={N} S={S}")
    assert np.array_equal(gst.view(np.uint32), os_[T - 1].view(np.uint32))
    for t in range(T):                                     # every frame's mask, bitwise
        assert np.array_equal(gm[t], om[t]), f"frame {t}: {(gm[t] != om[t]).sum()} mask pixels differ"


@pytest.mark.parametrize("prefilter,frame_warp", [((5, 1.0, 1), False), (None, True), ((5, 1.0, 1), True)])
def test_fullsize_paper_modes(cuda_lib, oracle_mod, prefilter, frame_warp, monkeypatch):
    """The bench's C4 launch configuration (32 x 1080p, N=4) with the paper's own
    preprocessing (NEXT-2) and/or frame-warp motion compensation (NEXT-3): every CTA of
    the persistent warp kernel walks ~20 tiles (plan-ring wrap, stream changes inside a
    CTA's range) and the streaming filter covers the whole batch.  Sampled streams against
    the oracle run as filter -> warp -> step with H = I (R34, R35)."""
    monkeypatch.delenv("DMSGM_KERNEL", raising=False)
    import torch
    dm = cuda_lib
    sample = [0, 13, 31]
    T = 3
    cfg = synth.config("C4", T=T)
    seq = synth.generate(cfg, streams=sample)
    S, H, W, N = cfg.S, cfg.H, cfg.W, cfg.N
    src = [sample.index(s) if s in sample else s % len(sample) for s in range(S)]
    pg, _ = params_pair(dm, oracle_mod, S)
    ctx = dm.Dmsgm(W, H, N, pg)
    if prefilter:
        ctx.set_prefilter(*prefilter)
    if frame_warp:
        ctx.set_motion(dm.DMSGM_MC_FRAME)
    frames = seq.frames if not prefilter else oracle_mod.prefilter_frames(seq.frames, *prefilter)
    if frame_warp:
        frames = oracle_mod.warp_frames(frames, seq.homographies)
        homs = np.broadcast_to(np.eye(3).reshape(9), seq.homographies.shape).copy()
    else:
        homs = seq.homographies
    o = oracle_mod.Oracle(W, H, N, params_pair(dm, oracle_mod, len(sample))[1])
    f = torch.empty((S, H, W), dtype=torch.uint8, device="cuda")
    m = torch.empty_like(f)
    for t in range(T):
        f.copy_(torch.from_numpy(seq.frames[t][src]))
        h = torch.from_numpy(np.ascontiguousarray(seq.homographies[t][src])).cuda()
        ctx.step(f, h, m)
        om = o.step(frames[t], homs[t])
        torch.cuda.synchronize()
        gm = m.cpu().numpy()
        ost = np.stack([o.get_state(j) for j in range(len(sample))])
        gst = np.stack([ctx.get_state(s) for s in sample])
        where = f"C4 prefilter={prefilter} frame_warp={frame_warp} t={t}"
        compare_state(gst, ost, where=where)
        compare_masks(gm[sample], om, frames[t], (ost[:, 0], ost[:, 1]), N, where=where)
    ctx.close()
    o.close()


def test_fullsize_warp_and_filter_kernels(cuda_lib, oracle_mod):
    """The stand-alone warp and filter kernels over the whole C4 batch (32 x 1080p, the
    bench's grid), every stream bitwise against the oracle."""
    import torch
    cfg = synth.config("C4", T=1)
    sample = [0, 9, 22]
    seq = synth.generate(cfg, streams=sample)
    S = cfg.S
    src = [sample.index(s) if s in sample else s % len(sample) for s in range(S)]
    fr = seq.frames[0][src]
    hs = np.ascontiguousarray(seq.homographies[0][src])
    f = torch.from_numpy(fr).cuda()
    out = torch.empty_like(f)
    cuda_lib.warp_frames(f, torch.from_numpy(hs).cuda(), out)
    torch.cuda.synchronize()
    want = oracle_mod.warp_frames(seq.frames[0], seq.homographies[0])
    got = out.cpu().numpy()
    for s in range(S):
        assert np.array_equal(got[s], want[src[s]]), f"warp stream {s}: {(got[s] != want[src[s]]).sum()} px differ"
    cuda_lib.prefilter(f, out, 5, 1.0, 1)
    torch.cuda.synchronize()
    want = oracle_mod.prefilter_frames(seq.frames[0], 5, 1.0, 1)
    got = out.cpu().numpy()
    for s in range(S):
        assert np.array_equal(got[s], want[src[s]]), f"filter stream {s}: {(got[s] != want[src[s]]).sum()} px differ"
