import sys, numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import synth, oracle
from paper_1702_05156_b200 import dmsgm as dm
from gpu_util import run_gpu, run_oracle, params_pair
for name, T, kw in [("C2", 300, {}), ("C3", 300, {}), ("C2", 300, dict(decay_var_thresh=100.0, decay_lambda=0.01))]:
    cfg = synth.config(name, T=T); seq = synth.generate(cfg)
    pg, po = params_pair(dm, oracle, cfg.S, **kw)
    gm, gs = run_gpu(dm, seq.frames, seq.homographies, cfg.N, pg, snapshot_every=25)
    om, os_ = run_oracle(oracle, seq.frames, seq.homographies, cfg.N, po, snapshot_every=25)
    nb = sum(int(np.sum(gs[t].view(np.uint32) != os_[t].view(np.uint32))) for t in gs)
    print(name, T, kw, "state values differing bitwise:", nb, "masks differing:", int(np.sum(gm != om)))
