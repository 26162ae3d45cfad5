"""Can the (ALU-bound) prefilter of frame t+1 overlap the (HBM-bound) step of frame t?
C4 ring, 32 streams: per iteration one dmsgm_prefilter launch and one dmsgm_step launch,
either on one stream (sequential, today's pipeline) or on two streams (prefilter t+1 on B
while step t runs on A; B waits for A's step t-1 so the pipeline stays one frame deep).
Run under DMSGM_STAGED_CTAS_PER_SM=2|3 and with a low-register filter build
(DMSGM_LIB_PATH) to see whether co-residency pays.  Prints one JSON line.

  DMSGM_STAGED_CTAS_PER_SM=2 DMSGM_LIB_PATH=ab/libpf_c4m3.so python scripts/pf_overlap.py
"""
from __future__ import annotations

import json
import os
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
    A = torch.cuda.current_stream()
    B = torch.cuda.Stream()
    cfg = synth.config("C4ring", S=32)
    ring, Hs = synth.generate_device(cfg, T=8, device="cuda:0")
    Hd = torch.from_numpy(np.ascontiguousarray(Hs)).cuda()
    masks = torch.empty_like(ring[0])
    filt = [torch.empty_like(ring[0]) for _ in range(2)]
    ctx = dm.Dmsgm(cfg.W, cfg.H, cfg.N, bench.method_params(dm, 32))
    K = 200
    res = {"ctas_per_sm": os.environ.get("DMSGM_STAGED_CTAS_PER_SM", "default"),
           "lib": os.environ.get("DMSGM_LIB_PATH", "default")}

    def seq(k):
        for i in range(k):
            dm.prefilter(ring[i % 8], filt[i % 2], 5, 1.0, 1, stream=A)
            ctx.step(filt[i % 2], Hd[i % 8], masks, A)

    def ovl(k):
        done = [torch.cuda.Event() for _ in range(2)]
        ready = [torch.cuda.Event() for _ in range(2)]
        with torch.cuda.stream(B):
            dm.prefilter(ring[0], filt[0], 5, 1.0, 1, stream=B)
            ready[0].record(B)
        for i in range(k):
            # B: the filter of frame i+1 into the other buffer, after step i-1 read it
            if i + 1 < k:
                if i >= 1:
                    B.wait_event(done[(i - 1) % 2])
                dm.prefilter(ring[(i + 1) % 8], filt[(i + 1) % 2], 5, 1.0, 1, stream=B)
                ready[(i + 1) % 2].record(B)
            A.wait_event(ready[i % 2])
            ctx.step(filt[i % 2], Hd[i % 8], masks, A)
            done[i % 2].record(A)

    for name, fn in (("sequential", seq), ("two_streams", ovl)):
        fn(10)
        torch.cuda.synchronize()
        torch.cuda._sleep(200_000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(A)
        fn(K)
        A.wait_stream(B)
        e1.record(A)
        e1.synchronize()
        res[name + "_us_per_frame"] = round(1000 * e0.elapsed_time(e1) / K, 2)
    # each kernel alone
    for name, fn in (("prefilter_only", lambda k: [dm.prefilter(ring[i % 8], filt[i % 2], 5, 1.0, 1, stream=A)
                                                   for i in range(k)]),
                     ("step_only", lambda k: [ctx.step(ring[i % 8], Hd[i % 8], masks, A) for i in range(k)])):
        fn(10)
        torch.cuda.synchronize()
        torch.cuda._sleep(200_000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(A)
        fn(K)
        e1.record(A)
        e1.synchronize()
        res[name + "_us"] = round(1000 * e0.elapsed_time(e1) / K, 2)
    ctx.close()
    print(json.dumps(res))


if __name__ == "__main__":
    main()
