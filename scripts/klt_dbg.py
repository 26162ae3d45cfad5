import sys
import numpy as np
import torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import paper_1702_05156_b200 as dm
import synth
from oracle import klt_oracle as K
cfg = synth.config("C4", T=2)
seq = synth.generate(cfg, streams=range(2))
frames = seq.frames
T, S, H, W = frames.shape
kp = dm.KltParams(num_streams=S); op = K.KltParams()
k = dm.Klt(W, H, kp)
cor = np.zeros((S, kp.max_corners, 2), np.int32); cnt = np.zeros(S, np.int32); refs = []
for s in range(S):
    c = K.good_features(frames[0, s], op); cor[s, :len(c)] = c; cnt[s] = len(c)
    refs.append(K.lk_track(frames[0, s], frames[1, s], c, op))
tr = torch.zeros((S, kp.max_corners, 2), dtype=torch.float32, device="cuda")
st = torch.zeros((S, kp.max_corners), dtype=torch.uint8, device="cuda")
k.track(torch.from_numpy(frames[0]).cuda(), torch.from_numpy(frames[1]).cuda(), torch.from_numpy(cor).cuda(), torch.from_numpy(cnt).cuda(), tr, st)
torch.cuda.synchronize()
for s in range(S):
    n = int(cnt[s]); out, ost = refs[s]
    g = tr[s, :n].cpu().numpy().astype(np.float64); gs = st[s, :n].cpu().numpy().astype(bool)
    Hinv = np.linalg.inv(seq.homographies[1, s].reshape(3, 3))
    c = cor[s, :n] + 0.5
    q = (Hinv @ np.c_[c, np.ones(n)].T).T; truth = q[:, :2] / q[:, 2:3]
    d = np.abs(g - out).max(1)
    print("stream", s, "n", n, "status diff", (gs != ost).sum(), "d>0.02:", (d > 0.02).sum(), "d>0.001:", (d > 0.001).sum(), "median d", np.nanmedian(d))
    for i in np.nonzero(d > 0.02)[0][:10]:
        print("  ", i, cor[s, i], "oracle", out[i], "gpu", g[i], "truth", truth[i], "oerr", np.abs(out[i]-truth[i]).max(), "gerr", np.abs(g[i]-truth[i]).max())
