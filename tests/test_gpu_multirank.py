"""The CUDA path under ranks: two processes on cuda:0 (the only GPU a test box has), each
with its own Dmsgm context over its weak shard of the streams, joined through a gloo
process group exactly as bench.py does under torchrun (shard.weak_shard, gather_digests,
max_over_ranks).  Streams are independent problems, so the per-stream digests (last mask +
final state, bitwise) of the sharded run must equal those of ONE process running the whole
batch through the CUDA path, and those of the oracle.  Both ranks step through
dmsgm_step_n graphs, the bench's timed path."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SPR = 3          # streams per rank
T = 6


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run_cuda(dm, frames, Hs, N, S):
    import torch
    T_, S_, H, W = frames.shape
    p = dm.Params(num_streams=S)
    ctx = dm.Dmsgm(W, H, N, p, device=0)
    f = torch.from_numpy(frames).cuda()
    h = torch.from_numpy(np.ascontiguousarray(Hs)).cuda()
    m = torch.zeros_like(f)
    ctx.step(f[0], h[0], m[0])                     # first step: initialises every stream
    ctx.step_n(T_ - 1, f[1:], h[1:], m[1:])       # then the graph path
    torch.cuda.synchronize()
    masks = m.cpu().numpy()
    states = np.stack([ctx.get_state(s) for s in range(S)])
    ctx.close()
    return masks, states


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK="0")
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    import paper_1702_05156_b200 as dm
    import synth
    from paper_1702_05156_b200.shard import env_rank, gather_digests, max_over_ranks, stream_digest, weak_shard

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    r, w, _ = env_rank()
    shard = weak_shard(r, w, SPR, local_rank=0)
    cfg = synth.config("C2", T=T, S=SPR * world)
    seq = synth.generate(cfg, streams=list(shard.streams))
    masks, states = _run_cuda(dm, seq.frames, seq.homographies, cfg.N, shard.num_streams)
    local_d = {s: stream_digest(masks[-1, j], states[j]) for j, s in enumerate(shard.streams)}
    merged = gather_digests(local_d)
    t = max_over_ranks(1.0 + rank)
    dist.barrier()
    if rank == 0:
        np.save(os.path.join(out_dir, "digests.npy"), np.array(sorted(merged.items()), dtype=object),
                allow_pickle=True)
        with open(os.path.join(out_dir, "tmax.txt"), "w") as f:
            f.write(repr(t))
    dist.destroy_process_group()


def test_two_ranks_on_one_gpu_equal_single_process(cuda_lib, oracle_mod, tmp_path):
    import torch.multiprocessing as mp

    import synth
    from paper_1702_05156_b200.shard import stream_digest
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    got = dict(np.load(tmp_path / "digests.npy", allow_pickle=True).tolist())
    assert float(open(tmp_path / "tmax.txt").read()) == 2.0
    cfg = synth.config("C2", T=T, S=SPR * world)
    seq = synth.generate(cfg)
    masks, states = _run_cuda(cuda_lib, seq.frames, seq.homographies, cfg.N, cfg.S)
    one = {s: stream_digest(masks[-1, s], states[s]) for s in range(cfg.S)}
    assert got == one, "sharded CUDA run differs from the single-process CUDA run"
    p = oracle_mod.OracleParams(num_streams=cfg.S)
    om, ofinal, _ = oracle_mod.run_sequence(seq.frames, seq.homographies, cfg.N, p)
    ref = {s: stream_digest(om[-1, s], ofinal[s]) for s in range(cfg.S)}
    assert got == ref, "sharded CUDA run differs from the oracle"
