"""N > 1 path on CPU: world-size-2 gloo process group (no GPU needed).

Checks the host logic bench.py uses under torchrun: the stream sharding covers every
stream exactly once, the timed value is the MAX over ranks, and -- because streams are
independent -- a sharded run (each rank its own streams, no data-path collective)
produces per-stream results bitwise identical to one process running the whole batch.
The per-rank work here is the CPU oracle, standing in for the device kernel.
"""
import os
import socket

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_functions():
    from paper_1702_05156_b200 import build
    build.build()
    from paper_1702_05156_b200.shard import strong_shard, weak_shard
    for world in (1, 2, 4, 8):
        w = [weak_shard(r, world, 32) for r in range(world)]
        assert [s.first_stream for s in w] == [32 * r for r in range(world)]
        assert all(s.num_streams == 32 for s in w)
        for total in (world, 32, 33, 64, 101):
            sh = [strong_shard(r, world, total) for r in range(world)]
            covered = [i for s in sh for i in s.streams]
            assert covered == list(range(total))
            assert max(s.num_streams for s in sh) - min(s.num_streams for s in sh) <= 1
    with pytest.raises(ValueError):
        weak_shard(2, 2, 4)
    with pytest.raises(ValueError):
        strong_shard(0, 4, 3)


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    import oracle
    import synth
    from paper_1702_05156_b200.shard import env_rank, gather_digests, max_over_ranks, stream_digest, weak_shard

    dist.init_process_group("gloo", rank=rank, world_size=world)
    r, w, local = env_rank()
    assert (r, w, local) == (rank, world, rank)
    shard = weak_shard(r, w, 3)
    cfg = synth.config("C2", T=4, S=3 * world)
    seq = synth.generate(cfg, streams=list(shard.streams))
    p = oracle.OracleParams(num_streams=shard.num_streams)
    masks, final, _ = oracle.run_sequence(seq.frames, seq.homographies, cfg.N, p)
    local_d = {s: stream_digest(masks[-1, j], final[j]) for j, s in enumerate(shard.streams)}
    merged = gather_digests(local_d)
    t = max_over_ranks(10.0 + rank)
    dist.barrier()
    if rank == 0:
        np.save(os.path.join(out_dir, "digests.npy"), np.array(sorted(merged.items()), dtype=object),
                allow_pickle=True)
        with open(os.path.join(out_dir, "tmax.txt"), "w") as f:
            f.write(repr(t))
    dist.destroy_process_group()


def test_two_rank_sharded_equals_single(tmp_path, oracle_mod):
    import torch.multiprocessing as mp

    import synth
    from paper_1702_05156_b200.shard import stream_digest
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    got = dict(np.load(tmp_path / "digests.npy", allow_pickle=True).tolist())
    assert float(open(tmp_path / "tmax.txt").read()) == 11.0          # MAX over ranks
    # reference: one process, the whole batch
    cfg = synth.config("C2", T=4, S=3 * world)
    seq = synth.generate(cfg)
    p = oracle_mod.OracleParams(num_streams=cfg.S)
    masks, final, _ = oracle_mod.run_sequence(seq.frames, seq.homographies, cfg.N, p)
    ref = {s: stream_digest(masks[-1, s], final[s]) for s in range(cfg.S)}
    assert got == ref
