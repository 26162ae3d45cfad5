"""Where does a short timed region lose time?  The C4 step as a CUDA graph of K steps
(dmsgm_step_n), timed between CUDA events after a full sync, with and without a spin
kernel queued ahead of the start event (so the graph launch is already enqueued when the
start timestamp is taken), for several K.  Prints one JSON object.

  python scripts/k_overhead.py > gpurun_out/k_overhead.json
"""
from __future__ import annotations

import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    import bench
    import paper_1702_05156_b200 as dm
    import synth
    torch.cuda.set_device(0)
    stream = torch.cuda.current_stream()
    cfg = synth.config("C4ring", S=32)
    ring, Hs = synth.generate_device(cfg, T=8, device="cuda:0")
    frames = ring.repeat(5, 1, 1, 1)
    del ring
    Hd = torch.from_numpy(np.ascontiguousarray(np.tile(Hs, (5, 1, 1)))).cuda()
    masks = torch.empty_like(frames)
    ctx = dm.Dmsgm(cfg.W, cfg.H, cfg.N, bench.method_params(dm, 32))
    for i in range(5):
        ctx.step(frames[i], Hd[i], masks[i], stream)
    res = {}
    for K in (1, 5, 20, 40):
        ctx.step_n(K, frames[:K], Hd[:K], masks[:K], stream)          # capture + run
        torch.cuda.synchronize()
        for pre in (0, 1):
            ts = []
            for rep in range(6):
                torch.cuda.synchronize()
                if pre:
                    torch.cuda._sleep(100_000)                           # ~50 us of spinning
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                ctx.step_n(K, frames[:K], Hd[:K], masks[:K], stream)
                e1.record(stream)
                e1.synchronize()
                ts.append(1000 * e0.elapsed_time(e1) / K)
            res[f"K{K}_pre{pre}"] = dict(us_per_step=[round(t, 2) for t in ts], median=round(statistics.median(ts), 2))
    # back-to-back replays without sync in between (steady state)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(11)]
    ev[0].record(stream)
    for k in range(10):
        ctx.step_n(40, frames, Hd, masks, stream)
        ev[k + 1].record(stream)
    ev[-1].synchronize()
    res["b2b_K40"] = [round(1000 * ev[k].elapsed_time(ev[k + 1]) / 40, 2) for k in range(10)]
    ctx.close()
    print(json.dumps(res))


if __name__ == "__main__":
    main()
