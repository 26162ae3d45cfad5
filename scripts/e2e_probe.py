"""PCIe probe: pinned H2D / D2H bandwidth alone and concurrently, and dmsgm_step_host per chunking."""
import os, sys, time, json
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

dev = torch.device("cuda", 0)
nb = 32 * 1920 * 1080
h = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
h2 = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
d = torch.empty(nb, dtype=torch.uint8, device=dev)
d2 = torch.empty(nb, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, n=20):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n
out = {}
out["h2d_GBs"] = nb / t(lambda: d.copy_(h, non_blocking=True)) / 1e9
out["d2h_GBs"] = nb / t(lambda: h2.copy_(d2, non_blocking=True)) / 1e9
def both():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    s1.synchronize(); s2.synchronize()
out["both_each_GBs"] = nb / t(both) / 1e9
import synth
import paper_1702_05156_b200 as dm
cfg = synth.config("C4ring")
frames, Hs = synth.generate_device(cfg, T=2, device="cuda:0")
hf = [frames[r].cpu().pin_memory() for r in range(2)]
hm = torch.empty_like(hf[0]).pin_memory()
hH = torch.from_numpy(np.ascontiguousarray(Hs)).pin_memory()
for chunks in (4, 8, 16, 32):
    os.environ["DMSGM_HOST_CHUNKS"] = str(chunks)
    ctx = dm.Dmsgm(cfg.W, cfg.H, cfg.N, dm.Params(num_streams=cfg.S))
    for i in range(3): ctx.step_host(hf[i % 2], hH[i % 2], hm)
    t0 = time.perf_counter(); n = 30
    for i in range(n): ctx.step_host(hf[i % 2], hH[i % 2], hm)
    dt = (time.perf_counter() - t0) / n
    out[f"step_host_chunks{chunks}_ms"] = dt * 1e3
    out[f"step_host_chunks{chunks}_fps"] = cfg.S / dt
    ctx.close()
print(json.dumps(out))
