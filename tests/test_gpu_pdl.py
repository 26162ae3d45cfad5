"""Stream-order contract of the step under programmatic dependent launch (include/dmsgm.h).

Every step launch may begin while the kernel before it on the stream drains; the step must
still see frames that kernel wrote.  Here a producer KERNEL (not a copy-engine transfer)
rewrites ONE frame buffer right before every step -- so a step that read its frame tile
before griddepcontrol.wait could see the previous frame -- in the three modes whose
kernel chains differ: plain steps, preprocessing (the context's filter kernel writes the
frames the step reads) and frame warping (the warp kernel does).  Results must equal the
oracle's bitwise.  dmsgm_step_n, whose steps load their first frame tile before the wait
(legal there: the frames are graph inputs), is checked the same way on a ring.
"""
import numpy as np
import pytest

import synth
from gpu_util import params_pair

pytestmark = pytest.mark.gpu


def _oracle_run(oracle_mod, frames, Hs, N, po, mode):
    T, S, H, W = frames.shape
    o = oracle_mod.Oracle(W, H, N, po)
    ident = np.broadcast_to(np.eye(3).reshape(9), Hs.shape[1:]).copy()
    masks = []
    for t in range(T):
        f = frames[t]
        h = Hs[t]
        if mode in ("prefilter", "frame+prefilter"):
            f = oracle_mod.prefilter_frames(f, 5, 1.0, 1)
        if mode in ("frame", "frame+prefilter"):
            f = oracle_mod.warp_frames(f, h)
            h = ident
        masks.append(o.step(np.ascontiguousarray(f), h))
    states = np.stack([o.get_state(s) for s in range(S)])
    o.close()
    return np.stack(masks), states


@pytest.mark.parametrize("mode", ["plain", "prefilter", "frame", "frame+prefilter"])
def test_producer_kernel_then_step(cuda_lib, oracle_mod, mode):
    import torch
    dm = cuda_lib
    cfg = synth.config("C2", T=24, S=3)
    seq = synth.generate(cfg)
    T, S, H, W = seq.frames.shape
    pg, po = params_pair(dm, oracle_mod, S)
    ctx = dm.Dmsgm(W, H, cfg.N, pg)
    if "prefilter" in mode:
        ctx.set_prefilter(5, 1.0, 1)
    if "frame" in mode:
        ctx.set_motion(dm.DMSGM_MC_FRAME)
    src = torch.from_numpy(seq.frames).cuda()
    hs = torch.from_numpy(seq.homographies).cuda()
    key = torch.zeros_like(src[0])
    fbuf = torch.empty_like(src[0])                   # ONE frame buffer, rewritten every step
    masks = torch.zeros_like(src)
    stream = torch.cuda.current_stream()
    for t in range(T):
        torch.bitwise_xor(src[t], key, out=fbuf)      # an elementwise kernel writes the frames
        ctx.step(fbuf, hs[t], masks[t], stream)
    torch.cuda.synchronize()
    gm = masks.cpu().numpy()
    gs = np.stack([ctx.get_state(s) for s in range(S)])
    ctx.close()
    om, os_ = _oracle_run(oracle_mod, seq.frames, seq.homographies, cfg.N, po, mode)
    assert np.array_equal(gm, om), f"{mode}: {(gm != om).sum()} mask pixels differ"
    assert np.array_equal(gs.view(np.uint32), os_.view(np.uint32)), f"{mode}: states differ"


def test_step_n_ring_early_frames(cuda_lib, oracle_mod):
    """dmsgm_step_n over a ring whose frames a kernel wrote just before the graph launch."""
    import torch
    dm = cuda_lib
    cfg = synth.config("C2", T=16, S=2)
    seq = synth.generate(cfg)
    T, S, H, W = seq.frames.shape
    pg, po = params_pair(dm, oracle_mod, S)
    ctx = dm.Dmsgm(W, H, cfg.N, pg)
    src = torch.from_numpy(seq.frames).cuda()
    hs = torch.from_numpy(seq.homographies).cuda()
    ring = torch.empty_like(src[:8])
    masks = torch.zeros_like(src)
    for half in range(2):
        torch.bitwise_xor(src[8 * half:8 * half + 8], torch.zeros_like(ring), out=ring)
        ctx.step_n(8, ring, hs[8 * half:8 * half + 8], masks[8 * half:8 * half + 8])
    torch.cuda.synchronize()
    gm = masks.cpu().numpy()
    gs = np.stack([ctx.get_state(s) for s in range(S)])
    ctx.close()
    om, os_ = _oracle_run(oracle_mod, seq.frames, seq.homographies, cfg.N, po, "plain")
    assert np.array_equal(gm, om)
    assert np.array_equal(gs.view(np.uint32), os_.view(np.uint32))


def test_host_async_after_device_steps(cuda_lib, oracle_mod):
    """dmsgm_step_host_async right after dmsgm_step on the same stream reads the state that
    step wrote (the async host path waits on the last device-side step)."""
    import torch
    dm = cuda_lib
    cfg = synth.config("C2", T=12, S=2)
    seq = synth.generate(cfg)
    T, S, H, W = seq.frames.shape
    pg, po = params_pair(dm, oracle_mod, S)
    ctx = dm.Dmsgm(W, H, cfg.N, pg)
    src = torch.from_numpy(seq.frames).cuda()
    hs = torch.from_numpy(seq.homographies).cuda()
    dmask = torch.zeros_like(src[0])
    hf = [torch.from_numpy(seq.frames[t]).pin_memory() for t in range(T)]
    hh = [torch.from_numpy(np.ascontiguousarray(seq.homographies[t])).pin_memory() for t in range(T)]
    hm = [torch.zeros((S, H, W), dtype=torch.uint8).pin_memory() for _ in range(T)]
    stream = torch.cuda.current_stream()
    ctx.step_host(hf[0], hh[0], hm[0], stream)        # sets up the host pipeline
    for t in range(1, T):
        if t % 3 == 1:
            ctx.step(src[t], hs[t], dmask, stream)     # device-side step ...
            hm[t].copy_(dmask.cpu())
        else:
            ctx.step_host_async(hf[t], hh[t], hm[t], stream)   # ... then host steps on its state
    torch.cuda.synchronize()
    gm = np.stack([m.numpy() for m in hm])
    gs = np.stack([ctx.get_state(s) for s in range(S)])
    ctx.close()
    om, os_ = _oracle_run(oracle_mod, seq.frames, seq.homographies, cfg.N, po, "plain")
    assert np.array_equal(gm, om)
    assert np.array_equal(gs.view(np.uint32), os_.view(np.uint32))


def test_host_staging_grows_with_band(cuda_lib, oracle_mod):
    """step_host staging sized at first use must grow when dmsgm_set_band makes
    the images taller (band -> whole frame)."""
    import torch
    dm = cuda_lib
    cfg = synth.config("C2", T=4, S=1)
    seq = synth.generate(cfg)
    T, S, H, W = seq.frames.shape
    N = cfg.N
    pg, po = params_pair(dm, oracle_mod, S)
    ctx = dm.Dmsgm(W, H, N, pg)
    rows = (H // N) // 3
    ctx.set_band(0, rows, 0)
    band = np.ascontiguousarray(seq.frames[0][:, :rows * N])
    hm = np.zeros_like(band)
    ctx.step_host(band, np.ascontiguousarray(seq.homographies[0]), hm)
    ctx.set_band(0, H // N, 0)                        # whole frame: 3x taller images
    masks = []
    for t in range(T):
        m = np.zeros((S, H, W), np.uint8)
        ctx.step_host(np.ascontiguousarray(seq.frames[t]), np.ascontiguousarray(seq.homographies[t]), m)
        masks.append(m)
    torch.cuda.synchronize()
    gs = np.stack([ctx.get_state(s) for s in range(S)])
    ctx.close()
    om, os_ = _oracle_run(oracle_mod, seq.frames, seq.homographies, N, po, "plain")
    assert np.array_equal(np.stack(masks), om)
    assert np.array_equal(gs.view(np.uint32), os_.view(np.uint32))
