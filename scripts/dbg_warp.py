import sys, numpy as np, torch
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import synth, oracle
from paper_1702_05156_b200 import dmsgm as dm
import test_gpu_warp as T
case = "zoom_rot"
rng = np.random.default_rng(sum(map(ord, case)))
W, H = 1920, 72
homs = [T._similarity(W, H, 1.0005, 0.05, 1.3, -0.7), T._similarity(W, H, 0.98, -2.0, -3, 2),
        synth.random_homography(rng, W, H, shift=4, rot_deg=3, zoom=0.05, persp=2e-5), T._similarity(W, H, 1.2, 0.0)]
Hs = np.stack(homs); S = len(Hs)
yy, xx = np.mgrid[0:H, 0:W]
frames = np.clip(120 + 90 * np.sin(xx / 5.0 + yy / 7.0) + rng.normal(0, 20, (S, H, W)), 0, 255).astype(np.uint8)
fin = torch.from_numpy(frames).cuda(); fout = torch.zeros_like(fin)
dm.warp_frames(fin, torch.from_numpy(Hs).cuda(), fout); torch.cuda.synchronize()
got = fout.cpu().numpy(); want = oracle.warp_frames(frames, Hs)
print("H2", Hs[2])
for s in range(S):
    ys, xs = np.nonzero(got[s] != want[s])
    for y, x in zip(ys, xs):
        print(s, "y", y, "x", x, "tile", x // 256, y // 16, "got", got[s, y, x], "want", want[s, y, x])
