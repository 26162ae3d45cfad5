import sys, numpy as np, torch
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import oracle
from paper_1702_05156_b200 import dmsgm as dm
for (W, H, S, dx) in [(100, 37, 3, 0.0), (100, 37, 3, 1.5), (256, 64, 2, 0.0), (512, 16, 1, 0.25), (512, 32, 1, 0.25)]:
    rng = np.random.default_rng(0)
    frames = rng.integers(0, 256, (S, H, W)).astype(np.uint8)
    Hs = np.tile(np.array([1, 0, dx, 0, 1, 0, 0, 0, 1.0]), (S, 1))
    pitch = (W + 15) // 16 * 16
    fin = torch.zeros((S, H, pitch), dtype=torch.uint8, device="cuda"); fin[..., :W] = torch.from_numpy(frames).cuda()
    fout = torch.full((S, H, pitch), 7, dtype=torch.uint8, device="cuda")
    dm.warp_frames(fin[..., :W], torch.from_numpy(Hs).cuda(), fout[..., :W]); torch.cuda.synchronize()
    got = fout[..., :W].cpu().numpy(); want = oracle.warp_frames(frames, Hs)
    d = got != want
    print(W, H, S, dx, "diff", d.sum(), "rows", sorted(set(np.nonzero(d)[1].tolist()))[:40], "cols", sorted(set(np.nonzero(d)[2].tolist()))[:10],
          "streams", sorted(set(np.nonzero(d)[0].tolist())))
    if d.sum():
        s, y, x = [v[0] for v in np.nonzero(d)]
        print("  first", s, y, x, "got", got[s, y, x], "want", want[s, y, x], "in", frames[s, y, x], "got row", got[s, y, :8], "want row", want[s, y, :8])
