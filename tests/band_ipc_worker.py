"""Two-process row-band run on ONE GPU through CUDA IPC (driven by tests/test_gpu_band.py).

Rank r (of 2) owns band r of a C2 sequence, opens its neighbour's state buffers and
sync words from IPC handles swapped over a gloo group (the same BandRank code torchrun
uses across GPUs), and steps T frames.  The parent then runs the whole frame in one
context and requires bitwise-equal masks and states.  Prints IPC-OK on success.
"""
import os
import socket
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
T = 8


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    import synth
    from paper_1702_05156_b200 import dmsgm
    from paper_1702_05156_b200.band import BandRank, band_rows, halo_for
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = synth.config("C2", T=T)
    seq = synth.generate(cfg)
    W, H, N = cfg.W, cfg.H, cfg.N
    bands = band_rows(H // N, world)
    halo = halo_for(W, H, N, seq.homographies.reshape(-1, 9), bands)
    br = BandRank(W, H, N, dmsgm.Params(num_streams=1), rank, world, halo, device=0, exchange="peer")
    b = br.band
    dev = torch.device("cuda", 0)
    pitch = (W + 15) // 16 * 16
    f = torch.zeros((1, b.rows * N, pitch), dtype=torch.uint8, device=dev)
    m = torch.zeros_like(f)
    masks = np.empty((T, b.rows * N, W), np.uint8)
    for t in range(T):
        f[0, :, :W] = torch.from_numpy(np.ascontiguousarray(seq.frames[t, 0, b.row0 * N:b.row1 * N])).to(dev)
        h = torch.from_numpy(np.ascontiguousarray(seq.homographies[t])).to(dev)
        br.step(f, h, m)
        torch.cuda.synchronize()
        masks[t] = m[0, :, :W].cpu().numpy()
    st = br.ctx.get_state(0)[:, b.row0:b.row1]
    status = br.ctx.get_status()
    np.savez(os.path.join(out, f"rank{rank}.npz"), masks=masks, state=st, status=status, row0=b.row0,
             row1=b.row1)
    dist.barrier()
    br.close()
    dist.destroy_process_group()


def main():
    import torch.multiprocessing as mp

    import synth
    from gpu_util import run_gpu
    from paper_1702_05156_b200 import dmsgm
    world = 2
    with tempfile.TemporaryDirectory() as out:
        mp.spawn(worker, args=(world, _port(), out), nprocs=world, join=True)
        cfg = synth.config("C2", T=T)
        seq = synth.generate(cfg)
        wm, ws = run_gpu(dmsgm, seq.frames, seq.homographies, cfg.N, dmsgm.Params(num_streams=1),
                         snapshot_every=T)
        N = cfg.N
        for r in range(world):
            d = np.load(os.path.join(out, f"rank{r}.npz"))
            assert int(d["status"]) == 0, f"rank {r} status {int(d['status'])}"
            r0, r1 = int(d["row0"]), int(d["row1"])
            assert np.array_equal(d["masks"], wm[:, 0, r0 * N:r1 * N]), f"rank {r} masks differ"
            ref = ws[T - 1][0][:, r0:r1]
            assert np.array_equal(d["state"].view(np.uint32), ref.view(np.uint32)), f"rank {r} state differs"
    print("IPC-OK")


if __name__ == "__main__":
    main()
