"""GPU motion estimation (include/dmsgm_klt.h) against the oracle
(oracle/klt_oracle.py), stage by stage and end to end, through the C ABI.

Bars: corners -- the same list in the same order (the scores are exact
integer tensors in fp64 on both sides); LK -- same status, tracked points within 0.02 px
(fp32 warp sums vs fp64 oracle); RANSAC -- fed the oracle's matches: the same per-iteration
inlier counts, the same inliers, and a homography whose image-corner reprojections agree
within 1e-3 px (Jacobi on A^T A vs the oracle's SVD); the whole chain on the synthetic
sequences -- within 0.05 px of the oracle's estimate and within 1 px of the generator's H_t
(the verdict's acceptance).
"""
import numpy as np
import pytest

import synth
from oracle import klt_oracle as K

pytestmark = pytest.mark.gpu


def _params(dm, S, **kw):
    return dm.KltParams(num_streams=S, **kw), K.KltParams(**kw)


def _proj(Hm, pts):
    q = (np.asarray(Hm).reshape(3, 3) @ np.c_[pts, np.ones(len(pts))].T).T
    return q[:, :2] / q[:, 2:3]


def _corner_err(H1, H2, W, H):
    c = np.array([[0, 0], [W, 0], [0, H], [W, H]], np.float64)
    return float(np.sqrt(((_proj(H1, c) - _proj(H2, c)) ** 2).sum(1)).max())


def _square_frames():
    f = np.zeros((3, 96, 128), np.uint8)
    f[0, 20:60, 30:90] = 255                                   # white rectangle
    y, x = np.mgrid[0:96, 0:128]
    f[1] = (((x // 8) + (y // 8)) % 2 * 255).astype(np.uint8)   # checkerboard: plateaus of equal scores
    f[2] = 77                                                   # constant: no corners
    return f


@pytest.mark.parametrize("case", ["C2", "C4", "shapes"])
def test_corners_equal_oracle(cuda_lib, case):
    import torch
    dm = cuda_lib
    if case == "shapes":
        frames = _square_frames()
    else:
        cfg = synth.config(case, T=1)
        frames = synth.generate(cfg, streams=range(3 if case == "C2" else 2)).frames[0]
    S, H, W = frames.shape
    kp, op = _params(dm, S, max_corners=300, min_distance=7.0)
    k = dm.Klt(W, H, kp)
    f = torch.from_numpy(frames).cuda()
    cor = torch.zeros((S, kp.max_corners, 2), dtype=torch.int32, device="cuda")
    cnt = torch.zeros(S, dtype=torch.int32, device="cuda")
    k.corners(f, cor, cnt)
    torch.cuda.synchronize()
    assert k.get_status() == 0
    for s in range(S):
        ref = K.good_features(frames[s], op)
        got = cor[s, :int(cnt[s])].cpu().numpy()
        assert np.array_equal(got, ref), f"stream {s}: {len(got)} vs {len(ref)} corners"
    k.close()


def _track_case(name, T=2, S=2):
    cfg = synth.config(name, T=T)
    seq = synth.generate(cfg, streams=range(S))
    return seq.frames, seq.homographies


def _true_next(corners, h):
    """Where the frame-(t-1) pixel centres of `corners` go in frame t under the generator's
    H_t (which maps frame t to frame t-1, R3)."""
    c = corners.astype(np.float64) + 0.5
    return _proj(np.linalg.inv(np.asarray(h).reshape(3, 3)), c)


@pytest.mark.parametrize("name", ["C2", "C3", "C4"])
def test_track_matches_oracle(cuda_lib, name):
    import torch
    dm = cuda_lib
    frames, hs = _track_case(name)
    T, S, H, W = frames.shape
    kp, op = _params(dm, S)
    k = dm.Klt(W, H, kp)
    cor = np.zeros((S, kp.max_corners, 2), np.int32)
    cnt = np.zeros(S, np.int32)
    refs = []
    for s in range(S):
        c = K.good_features(frames[0, s], op)
        cor[s, :len(c)] = c
        cnt[s] = len(c)
        refs.append(K.lk_track(frames[0, s], frames[1, s], c, op))
    prev = torch.from_numpy(frames[0]).cuda()
    nxt = torch.from_numpy(frames[1]).cuda()
    tr = torch.zeros((S, kp.max_corners, 2), dtype=torch.float32, device="cuda")
    st = torch.zeros((S, kp.max_corners), dtype=torch.uint8, device="cuda")
    k.track(prev, nxt, torch.from_numpy(cor).cuda(), torch.from_numpy(cnt).cuda(), tr, st)
    torch.cuda.synchronize()
    for s in range(S):
        n = int(cnt[s])
        out, ost = refs[s]
        gst = st[s, :n].cpu().numpy().astype(bool)
        gtr = tr[s, :n].cpu().numpy().astype(np.float64)
        assert np.array_equal(gst, ost), f"stream {s}: status differs on {(gst != ost).sum()} of {n}"
        d = np.abs(gtr - out).max(axis=1)
        far = ost & ~(d < 0.02)
        # A coarse pyramid level can hold several minima of the LK residual for a periodic
        # texture (level 5 of a 1080p frame is 60x33 px under a 20-px window); there the
        # rounding order may pick a different one, and the track lands 2^L periods away.
        # Allowed for <= 1 % of the points, and only where one of the two tracks is such a
        # wrong minimum (> 8 px from the true motion; RANSAC rejects it as an outlier).
        truth = _true_next(cor[s, :n], hs[1, s])
        wrong = (np.abs(out - truth).max(axis=1) > 8) | (np.abs(gtr - truth).max(axis=1) > 8)
        assert far.sum() <= max(1, 0.01 * ost.sum()), f"stream {s}: {far.sum()} of {ost.sum()} tracks differ"
        assert wrong[far].all(), f"stream {s}: tracks differ by up to {d[far].max()} px without a wrong minimum"
        print(f"{name} stream {s}: {ost.sum()} tracked, median |gpu - oracle| {np.median(d[ost]):.2e} px, "
              f"{far.sum()} on different minima")
    k.close()


def test_track_known_shift(cuda_lib):
    """Content shifted by (+3, -2) px: every tracked interior corner moves by it."""
    import torch
    dm = cuda_lib
    cfg = synth.config("C3", T=1)
    a = synth.generate(cfg).frames[0, 0]
    b = np.zeros_like(a)
    b[0:478, 3:] = a[2:480, :-3]                      # b(x, y) = a(x - 3, y + 2)
    kp, op = _params(dm, 1)
    k = dm.Klt(640, 480, kp)
    c = K.good_features(a, op)
    c = c[(c[:, 0] > 30) & (c[:, 0] < 610) & (c[:, 1] > 30) & (c[:, 1] < 450)]
    cor = np.zeros((1, kp.max_corners, 2), np.int32)
    cor[0, :len(c)] = c
    tr = torch.zeros((1, kp.max_corners, 2), dtype=torch.float32, device="cuda")
    st = torch.zeros((1, kp.max_corners), dtype=torch.uint8, device="cuda")
    k.track(torch.from_numpy(a[None]).cuda(), torch.from_numpy(b[None]).cuda(), torch.from_numpy(cor).cuda(),
            torch.tensor([len(c)], dtype=torch.int32, device="cuda"), tr, st)
    torch.cuda.synchronize()
    ok = st[0, :len(c)].cpu().numpy().astype(bool)
    flow = tr[0, :len(c)].cpu().numpy()[ok] - (c[ok] + 0.5)
    assert ok.mean() > 0.95
    assert np.abs(np.median(flow, axis=0) - [3.0, -2.0]).max() < 0.02
    k.close()


def _oracle_matches(frames, op):
    """The oracle's matches for a frame pair (src = frame-t point, dst = frame-(t-1) centre)."""
    c = K.good_features(frames[0], op)
    out, st = K.lk_track(frames[0], frames[1], c, op)
    return out[st], c[st].astype(np.float64) + 0.5


def test_ransac_matches_oracle(cuda_lib):
    import torch
    dm = cuda_lib
    rng = np.random.default_rng(7)
    sets = []
    # (a) SPEC S:310: 40 exact + 10 outliers; (b) the C2 / C4 oracle matches
    Hm = np.array([[1.01, 0.02, 3.0], [-0.015, 0.99, -2.0], [1e-4, -5e-5, 1.0]])
    src = rng.uniform(0, 320, (50, 2))
    dst = _proj(Hm, src)
    dst[rng.choice(50, 10, replace=False)] += rng.uniform(20, 60, (10, 2))
    sets.append((src, dst))
    for name in ("C2", "C4"):
        frames, _ = _track_case(name, S=1)
        sets.append(_oracle_matches(frames[:, 0], K.KltParams()))
    S = len(sets)
    kp, op = _params(dm, S)
    M = kp.max_corners
    k = dm.Klt(320, 240, kp)
    src = np.zeros((S, M, 2))
    dst = np.zeros((S, M, 2))
    cnt = np.zeros(S, np.int32)
    for s, (a, b) in enumerate(sets):
        src[s, :len(a)], dst[s, :len(b)], cnt[s] = a, b, len(a)
    Hg = torch.zeros((S, 9), dtype=torch.float64, device="cuda")
    inl = torch.zeros((S, M), dtype=torch.uint8, device="cuda")
    itc = torch.zeros((S, kp.ransac_iters), dtype=torch.int32, device="cuda")
    ok = torch.zeros(S, dtype=torch.int32, device="cuda")
    k.ransac(torch.from_numpy(src).cuda(), torch.from_numpy(dst).cuda(), torch.from_numpy(cnt).cuda(), Hg, inl, itc, ok)
    torch.cuda.synchronize()
    for s, (a, b) in enumerate(sets):
        Ho, io, co = K.ransac(a, b, op)
        n = len(a)
        assert np.array_equal(itc[s].cpu().numpy(), co), f"set {s}: per-iteration inlier counts differ"
        assert np.array_equal(inl[s, :n].cpu().numpy().astype(bool), io)
        assert int(ok[s]) == int(io.sum())
        assert _corner_err(Hg[s].cpu().numpy(), Ho, 320, 240) < 1e-3
    k.close()


@pytest.mark.parametrize("name,S,T,truth,thresh", [("C2", 2, 4, True, 3.0), ("C3", 1, 3, True, 3.0),
                                                   ("C4", 3, 2, False, 3.0), ("C4", 3, 2, True, 1.0),
                                                   ("C1", 1, 3, False, 3.0)])
def test_estimate_end_to_end(cuda_lib, name, S, T, truth, thresh):
    """The whole chain on the GPU (one dmsgm_klt_estimate per frame pair) vs the oracle's
    chain (within 0.1 px at the image corners) and vs the generator's H_t (within 1 px).
    Not checked against H_t: C1 (a 64x48 frame holds ~20 corners, the fit extrapolates
    to its corners: 1.7 px on both sides) and C4 at the paper's 3-px RANSAC threshold
    (OpenCV's default): foreground objects moving < 3 px/frame relative to the camera
    then count as inliers and bias the fit (up to 1.3 px at the 1080p corners, both sides);
    at 1 px the C4 corners are within 0.15 px."""
    import torch
    dm = cuda_lib
    cfg = synth.config(name, T=T)
    seq = synth.generate(cfg, streams=range(S))
    W, H = cfg.W, cfg.H
    kp, op = _params(dm, S, ransac_thresh=thresh)
    k = dm.Klt(W, H, kp)
    f = torch.from_numpy(seq.frames).cuda()
    Hg = torch.zeros((S, 9), dtype=torch.float64, device="cuda")
    ok = torch.zeros(S, dtype=torch.int32, device="cuda")
    for t in range(1, T):
        k.estimate(f[t - 1], f[t], Hg, ok)
        torch.cuda.synchronize()
        for s in range(S):
            Ho, det = K.estimate(seq.frames[t - 1, s], seq.frames[t, s], op)
            hg = Hg[s].cpu().numpy()
            # the inlier sets may differ by the few tracks on different LK minima (see above)
            assert abs(int(ok[s]) - int(det["inliers"].sum())) <= max(3, 0.02 * det["inliers"].sum())
            e_o, e_t = _corner_err(hg, Ho, W, H), _corner_err(hg, seq.homographies[t, s], W, H)
            print(f"{name} t={t} s={s}: inliers {int(ok[s])}, |H_gpu - H_oracle| {e_o:.2e} px, "
                  f"|H_gpu - H_t| {e_t:.3f} px at the image corners")
            assert e_o < 0.1, (t, s, e_o)
            assert e_t < 1.0 or not truth, (t, s, e_t)
    k.close()


def test_estimated_homographies_drive_the_step(cuda_lib):
    """The loop the paper's pipeline closes (App. F then App. E): homographies estimated on the
    GPU from the frames feed dmsgm_step; the masks' quality against the generator's ground
    truth matches that of the true homographies (SPEC S:453 moving-object criteria)."""
    import torch
    dm = cuda_lib
    cfg = synth.config("C2", T=40, S=2)
    seq = synth.generate(cfg, with_gt=True)
    T, S, H, W = seq.frames.shape
    k = dm.Klt(W, H, dm.KltParams(num_streams=S))
    f = torch.from_numpy(seq.frames).cuda()
    Ht = torch.from_numpy(seq.homographies).cuda()
    res = {}
    for mode in ("estimated", "true"):
        ctx = dm.Dmsgm(W, H, cfg.N, dm.Params(num_streams=S))
        m = torch.zeros_like(f)
        He = torch.zeros((S, 9), dtype=torch.float64, device="cuda")
        for t in range(T):
            if mode == "estimated" and t > 0:
                k.estimate(f[t - 1], f[t], He)
                ctx.step(f[t], He, m[t])
            else:
                ctx.step(f[t], Ht[t], m[t])
        torch.cuda.synchronize()
        gm = m[10:].cpu().numpy() > 0
        gt = seq.gt[10:] > 0
        res[mode] = (gm[gt].mean(), gm[~gt].mean())
        ctx.close()
    k.close()
    (cov_e, fp_e), (cov_t, fp_t) = res["estimated"], res["true"]
    assert cov_e >= cov_t - 0.02 and fp_e <= fp_t + 0.005, res
