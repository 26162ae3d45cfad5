"""Time dmsgm_klt_estimate (+ the step it feeds) on a bench ring: CUDA events, one GPU."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1702_05156_b200 as dm  # noqa: E402
import synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4ring"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
cfg = synth.config(name)
frames, Hs = synth.generate_device(cfg, T=8, device="cuda:0")
S, H, W = cfg.S, cfg.H, cfg.W
k = dm.Klt(W, H, dm.KltParams(num_streams=S))
He = torch.zeros((S, 9), dtype=torch.float64, device="cuda")
ok = torch.zeros(S, dtype=torch.int32, device="cuda")
st = torch.cuda.current_stream()
for i in range(3):
    k.estimate(frames[i % 8], frames[(i + 1) % 8], He, ok)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for i in range(reps):
    k.estimate(frames[i % 7], frames[i % 7 + 1], He, ok)
e1.record(st)
e1.synchronize()
ms = e0.elapsed_time(e1) / reps
# consecutive pairs through dmsgm_klt_estimate_seq (frames 0..7 of the ring, then 7 -> 0: a
# continuous motion, the ring is periodic)
for i in range(3):
    k.estimate_seq(frames[i % 8], frames[(i + 1) % 8], He, ok)
e0.record(st)
for i in range(3, 3 + reps):
    k.estimate_seq(frames[i % 8], frames[(i + 1) % 8], He, ok)
e1.record(st)
e1.synchronize()
ms_seq = e0.elapsed_time(e1) / reps
print(json.dumps({"config": name, "streams": S, "ms_per_estimate": ms, "frames_per_s": S / (ms / 1e3),
                  "ms_per_estimate_seq": ms_seq, "frames_per_s_seq": S / (ms_seq / 1e3),
                  "inliers_min": int(ok.min()), "status": k.get_status(), "levels": k.levels}))
