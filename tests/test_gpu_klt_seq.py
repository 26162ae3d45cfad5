"""dmsgm_klt_estimate_seq (include/dmsgm_klt.h): the estimate of consecutive frame pairs that
reuses the corners and pyramid of the previous call's `next` frame -- bitwise the H and
inlier counts of dmsgm_klt_estimate on every pair (it runs the same kernels on the same
bytes, only scheduled differently), including jumps (prev not the cached frame), resets,
interleaved stateless calls, and ragged / unaligned frames that take the pyramid kernel's
per-pixel path; and the pyramid itself against the oracle through the whole chain."""
import numpy as np
import pytest

import synth
from oracle import klt_oracle as K

pytestmark = pytest.mark.gpu


def _proj(Hm, pts):
    q = (np.asarray(Hm).reshape(3, 3) @ np.c_[pts, np.ones(len(pts))].T).T
    return q[:, :2] / q[:, 2:3]


def _corner_err(H1, H2, W, H):
    c = np.array([[0, 0], [W, 0], [0, H], [W, H]], np.float64)
    return float(np.sqrt(((_proj(H1, c) - _proj(H2, c)) ** 2).sum(1)).max())


def _frames(name, T, S, crop=None, pad=0):
    """uint8 CUDA frames [T][S][H][W] (optionally cropped to crop = (W, H), inside rows of
    W + pad bytes: a pitch that is not a multiple of 16 when pad is odd)."""
    import torch
    cfg = synth.config(name, T=T)
    f = synth.generate(cfg, streams=range(S)).frames
    if crop:
        f = np.ascontiguousarray(f[:, :, :crop[1], :crop[0]])
    T_, S_, H, W = f.shape
    buf = torch.zeros((T_, S_, H, W + pad), dtype=torch.uint8, device="cuda")
    buf[..., :W] = torch.from_numpy(f).cuda()
    return f, buf[..., :W]


@pytest.mark.parametrize("name,S,crop,pad", [("C2", 2, None, 0), ("C2", 2, (310, 230), 0), ("C2", 1, (310, 230), 11),
                                             ("C4", 2, None, 0)])
def test_seq_equals_stateless(cuda_lib, name, S, crop, pad):
    import torch
    dm = cuda_lib
    T = 5 if name == "C2" else 4
    host, f = _frames(name, T, S, crop, pad)
    H, W = host.shape[2:]
    k_seq = dm.Klt(W, H, dm.KltParams(num_streams=S))
    k_one = dm.Klt(W, H, dm.KltParams(num_streams=S))
    Hs = torch.zeros((S, 9), dtype=torch.float64, device="cuda")
    H1 = torch.zeros_like(Hs)
    oks = torch.zeros(S, dtype=torch.int32, device="cuda")
    ok1 = torch.zeros_like(oks)
    pairs = [(t - 1, t) for t in range(1, T)]            # consecutive: prev cached after the first
    pairs += [(0, 2), (2, 3)]                             # a jump (prev not cached), then continue
    for (a, b) in pairs:
        k_seq.estimate_seq(f[a], f[b], Hs, oks)
        k_one.estimate(f[a], f[b], H1, ok1)
        torch.cuda.synchronize()
        assert torch.equal(Hs, H1) and torch.equal(oks, ok1), (a, b, (Hs - H1).abs().max().item())
    # a stateless call on the same context drops the cache; seq_reset too
    k_seq.estimate(f[2], f[3], Hs, oks)
    k_seq.estimate_seq(f[3], f[4 % T], Hs, oks)
    k_one.estimate(f[3], f[4 % T], H1, ok1)
    torch.cuda.synchronize()
    assert torch.equal(Hs, H1) and torch.equal(oks, ok1)
    k_seq.seq_reset()
    k_seq.estimate_seq(f[4 % T], f[0], Hs, oks)
    k_one.estimate(f[4 % T], f[0], H1, ok1)
    torch.cuda.synchronize()
    assert torch.equal(Hs, H1) and torch.equal(oks, ok1)
    k_seq.close()
    k_one.close()


@pytest.mark.parametrize("crop,pad", [((310, 230), 0), ((310, 230), 11), ((333, 241), 3)])
def test_ragged_frames_match_oracle(cuda_lib, crop, pad):
    """Frames whose level-1 width is not a multiple of 8 (byte stores) and rows that are not
    16-byte aligned (the per-pixel level-1 path): the chain against the oracle's, which builds
    its own pyramid (R39), within the end-to-end test's 0.1 px at the image corners."""
    import torch
    dm = cuda_lib
    S = 2
    host, f = _frames("C2", 3, S, crop, pad)
    H, W = host.shape[2:]
    k = dm.Klt(W, H, dm.KltParams(num_streams=S))
    Hg = torch.zeros((S, 9), dtype=torch.float64, device="cuda")
    ok = torch.zeros(S, dtype=torch.int32, device="cuda")
    for t in (1, 2):
        k.estimate_seq(f[t - 1], f[t], Hg, ok)
        torch.cuda.synchronize()
        for s in range(S):
            Ho, det = K.estimate(host[t - 1, s], host[t, s], K.KltParams())
            assert abs(int(ok[s]) - int(det["inliers"].sum())) <= max(3, 0.02 * det["inliers"].sum())
            e = _corner_err(Hg[s].cpu().numpy(), Ho, W, H)
            assert e < 0.1, (t, s, e)
    k.close()


def test_outputs_stay_in_bounds(cuda_lib):
    """No KLT entry point writes past its outputs (the pool's compute-sanitizer is closed, see
    tests/test_gpu_sanitizer.py): every output is a view into a larger buffer filled with a
    canary byte; after corners / track / ransac / estimate / estimate_seq on ragged frames the
    bytes around each view are unchanged."""
    import torch
    dm = cuda_lib
    S = 2
    host, f = _frames("C2", 3, S, (310, 230), 11)
    H, W = host.shape[2:]
    kp = dm.KltParams(num_streams=S)
    M = kp.max_corners
    k = dm.Klt(W, H, kp)
    CAN = 0xA5

    def guarded(shape, dtype):
        n = int(np.prod(shape)) * torch.tensor([], dtype=dtype).element_size()
        raw = torch.full((n + 2048,), CAN, dtype=torch.uint8, device="cuda")
        return raw, raw[1024:1024 + n].view(dtype).view(shape)

    def intact(raw, n):
        r = raw.cpu().numpy()
        return (r[:1024] == CAN).all() and (r[1024 + n:] == CAN).all()

    outs = {}
    for name, shape, dtype in [("cor", (S, M, 2), torch.int32), ("cnt", (S,), torch.int32),
                               ("tr", (S, M, 2), torch.float32), ("st", (S, M), torch.uint8),
                               ("H", (S, 9), torch.float64), ("ok", (S,), torch.int32),
                               ("inl", (S, M), torch.uint8), ("itc", (S, kp.ransac_iters), torch.int32)]:
        outs[name] = guarded(shape, dtype)
    o = {n: v[1] for n, v in outs.items()}
    k.corners(f[0], o["cor"], o["cnt"])
    k.track(f[0], f[1], o["cor"], o["cnt"], o["tr"], o["st"])
    # matches from the tracked points (host-side compaction, as the oracle's chain does)
    torch.cuda.synchronize()
    src = np.zeros((S, M, 2)); dst = np.zeros((S, M, 2)); mc = np.zeros(S, np.int32)
    for s in range(S):
        n = int(o["cnt"][s]); ok = o["st"][s, :n].cpu().numpy().astype(bool)
        src[s, :ok.sum()] = o["tr"][s, :n].cpu().numpy()[ok]
        dst[s, :ok.sum()] = o["cor"][s, :n].cpu().numpy()[ok] + 0.5
        mc[s] = ok.sum()
    k.ransac(torch.from_numpy(src).cuda(), torch.from_numpy(dst).cuda(), torch.from_numpy(mc).cuda(), o["H"],
             o["inl"], o["itc"], o["ok"])
    k.estimate(f[0], f[1], o["H"], o["ok"])
    k.estimate_seq(f[1], f[2], o["H"], o["ok"])
    k.estimate_seq(f[2], f[0], o["H"], o["ok"])
    torch.cuda.synchronize()
    for name, (raw, view) in outs.items():
        assert intact(raw, view.numel() * view.element_size()), name
    assert k.get_status() == 0
    k.close()
