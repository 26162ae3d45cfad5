"""Small invocations of the frame-warp, prefilter and step kernels (every block size, both
step kernels, bit-packed masks) and of the homography estimation, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck): python scripts/sanitize_kernels.py"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth                                        # noqa: E402
from paper_1702_05156_b200 import dmsgm as dm       # noqa: E402
from paper_1702_05156_b200 import klt as kl         # noqa: E402

rng = np.random.default_rng(3)
S, H, W = 3, 100, 700                               # ragged tiles, several tiles per CTA
fr = torch.from_numpy(rng.integers(0, 256, (S, H, W), dtype=np.uint8)).cuda()
hs = np.stack([synth.random_homography(rng, W, H, shift=5, rot_deg=2, zoom=0.02, persp=1e-5) for _ in range(S)])
hs[1] = [1, 0, -40.5, 0, 1, 7.25, 0, 0, 1]          # border tiles far outside the frame
out = torch.empty_like(fr)
dm.warp_frames(fr, torch.from_numpy(hs).cuda(), out)
dm.prefilter(fr, out, 5, 1.0, 1)
cfg = synth.config("C2", T=3, S=2)
seq = synth.generate(cfg)
p = dict(theta_s=4.0, theta_d=4.0, var_init=255.0, age_cap=30.0, var_floor_match=0.1, var_floor_classify=0.25,
         decay_lambda=0.001, decay_var_thresh=2500.0, num_streams=cfg.S)
for mode in (dm.DMSGM_MC_MODELS, dm.DMSGM_MC_FRAME):
    ctx = dm.Dmsgm(cfg.W, cfg.H, cfg.N, dm.Params(**p))
    ctx.set_motion(mode)
    if mode == dm.DMSGM_MC_FRAME:
        ctx.set_prefilter(5, 1.0, 1)
    f = torch.from_numpy(seq.frames).cuda()
    h = torch.from_numpy(seq.homographies).cuda()
    m = torch.zeros_like(f)
    for t in range(cfg.T):
        ctx.step(f[t], h[t], m[t])
    ctx.close()
# every block size (staged kernels for N = 1, 2, 4, 8; the register-path kernel for N = 16
# and, forced, for N = 4) on random near-identity motion
import os                                            # noqa: E402
for N, generic in [(1, False), (2, False), (8, False), (16, False), (4, True)]:
    if generic:
        os.environ["DMSGM_KERNEL"] = "generic"
    Wn, Hn, Sn = 16 * 17, 16 * 5, 2
    pn = dict(p, num_streams=Sn)
    ctx = dm.Dmsgm(Wn, Hn, N, dm.Params(**pn))
    f = torch.from_numpy(rng.integers(0, 256, (3, Sn, Hn, Wn), dtype=np.uint8)).cuda()
    h = torch.from_numpy(np.stack([[synth.random_homography(rng, Wn, Hn, shift=3, rot_deg=1, zoom=0.01, persp=1e-5)
                                    for _ in range(Sn)] for _ in range(3)])).cuda()
    m = torch.zeros_like(f)
    for t in range(3):
        ctx.step(f[t], h[t], m[t])
    ctx.close()
    os.environ.pop("DMSGM_KERNEL", None)
# bit-packed masks (DMSGM_MASK_BITS, staged N = 4 and 8)
for N in (4, 8):
    Wn, Hn, Sn = 32 * N * 3, 9 * N, 2                # 9 block rows: a ragged tile row
    ctx = dm.Dmsgm(Wn, Hn, N, dm.Params(**dict(p, num_streams=Sn)))
    ctx.set_mask_format(dm.DMSGM_MASK_BITS)
    f = torch.from_numpy(rng.integers(0, 256, (3, Sn, Hn, Wn), dtype=np.uint8)).cuda()
    h = torch.from_numpy(np.stack([[synth.random_homography(rng, Wn, Hn, shift=3, rot_deg=1, zoom=0.01, persp=1e-5)
                                    for _ in range(Sn)] for _ in range(3)])).cuda()
    m = torch.zeros((3, Sn, Hn, (Wn + 7) // 8), dtype=torch.uint8, device="cuda")
    for t in range(3):
        ctx.step(f[t], h[t], m[t])
    ctx.close()
# homography estimation (NEXT-4): corners, pyramid, LK, RANSAC, refit on a shifted texture
Wk, Hk, Sk = 320, 240, 2
yy, xx = np.mgrid[0:Hk + 8, 0:Wk + 8]
tex = (120 + 60 * np.sin(xx / 5.0) * np.cos(yy / 7.0) + rng.normal(0, 8, xx.shape)).clip(0, 255).astype(np.uint8)
prev = torch.from_numpy(np.stack([tex[4:4 + Hk, 4:4 + Wk]] * Sk).copy()).cuda()
nxt = torch.from_numpy(np.stack([tex[2:2 + Hk, 7:7 + Wk]] * Sk).copy()).cuda()
klt = kl.Klt(Wk, Hk, kl.KltParams(num_streams=Sk))
Hk_out = torch.zeros((Sk, 9), dtype=torch.float64, device="cuda")
klt.estimate(prev, nxt, Hk_out)
klt.close()
torch.cuda.synchronize()
print("sanitize run ok")
