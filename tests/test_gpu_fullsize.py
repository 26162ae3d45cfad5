"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

C4: 32 streams of 1920x1080, N=4; C5: 64 streams of 3840x2160, N=8.  The GPU runs the
whole batch (same grid as the bench); the oracle recomputes a sample of streams in full
(streams are independent, so a stream's result does not depend on the rest of the batch;
test_batch_invariance pins that).  Non-sampled streams carry copies of sampled content.
"""
import numpy as np
import pytest

import synth
from gpu_util import compare_masks, compare_state, params_pair

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.mark.parametrize("name,T,sample", [("C4", 3, [0, 17, 31]), ("C5", 2, [5, 63])])
def test_fullsize_sampled_streams(cuda_lib, oracle_mod, name, T, sample, monkeypatch):
    monkeypatch.delenv("DMSGM_KERNEL", raising=False)       # the bench's kernel
    import torch
    dm = cuda_lib
    cfg = synth.config(name, T=T)
    seq = synth.generate(cfg, streams=sample)
    S, H, W, N = cfg.S, cfg.H, cfg.W, cfg.N
    src = [sample.index(s) if s in sample else s % len(sample) for s in range(S)]
    pg, po = params_pair(dm, oracle_mod, S)
    ctx = dm.Dmsgm(W, H, N, pg)
    f = torch.empty((S, H, W), dtype=torch.uint8, device="cuda")
    m = torch.empty_like(f)
    o_params = params_pair(dm, oracle_mod, len(sample))[1]
    o = oracle_mod.Oracle(W, H, N, o_params)
    for t in range(T):
        f.copy_(torch.from_numpy(seq.frames[t][src]))
        h = torch.from_numpy(np.ascontiguousarray(seq.homographies[t][src])).cuda()
        ctx.step(f, h, m)
        om = o.step(seq.frames[t], seq.homographies[t])
        torch.cuda.synchronize()
        gm = m.cpu().numpy()
        ost = np.stack([o.get_state(j) for j in range(len(sample))])
        gst = np.stack([ctx.get_state(s) for s in sample])
        compare_state(gst, ost, where=f"{name} t={t}")
        compare_masks(gm[sample], om, seq.frames[t], (ost[:, 0], ost[:, 1]), N, where=f"{name} t={t}")
    ctx.close()
    o.close()
