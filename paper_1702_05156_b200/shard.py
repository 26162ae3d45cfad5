"""Multi-GPU plumbing: stream sharding across ranks (one process per GPU).

Streams are independent problems, so the path shards with no
data-path collective: rank r of W owns its own streams, context, state, frames and
masks.  The only collectives are outside the timed kernels: a barrier around the
timed region, a MAX all-reduce of the per-rank device time, and (for checks) a gather
of per-stream checksums.  torch.distributed is used as plumbing only (NCCL on GPUs,
gloo on CPU for the tests).
"""
from __future__ import annotations

import hashlib
import os
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    local_rank: int
    first_stream: int      # global index of this rank's first stream
    num_streams: int       # streams this rank owns

    @property
    def streams(self) -> range:
        return range(self.first_stream, self.first_stream + self.num_streams)


def env_rank():
    """(rank, world, local_rank) from the torchrun environment (defaults: single process)."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def weak_shard(rank: int, world: int, streams_per_rank: int, local_rank: int | None = None) -> Shard:
    """Weak scaling: every rank runs `streams_per_rank` streams, rank r owns
    global streams [r*S, (r+1)*S) -- per-GPU work is fixed as the GPU count grows."""
    if world < 1 or not 0 <= rank < world or streams_per_rank < 1:
        raise ValueError("bad shard arguments")
    return Shard(rank, world, rank if local_rank is None else local_rank, rank * streams_per_rank,
                 streams_per_rank)


def strong_shard(rank: int, world: int, total_streams: int, local_rank: int | None = None) -> Shard:
    """Strong scaling: a fixed batch of `total_streams` split contiguously, as evenly as
    possible (the first total % world ranks get one more stream)."""
    if world < 1 or not 0 <= rank < world or total_streams < world:
        raise ValueError("bad shard arguments")
    base, extra = divmod(total_streams, world)
    first = rank * base + min(rank, extra)
    return Shard(rank, world, rank if local_rank is None else local_rank, first, base + (1 if rank < extra else 0))


def max_over_ranks(value: float, device=None) -> float:
    """MAX all-reduce of a per-rank scalar (e.g. the timed region's device milliseconds)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def stream_digest(mask: np.ndarray, state: np.ndarray) -> str:
    """A short digest of one stream's mask and model state (bitwise)."""
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(mask).tobytes())
    h.update(np.ascontiguousarray(state, np.float32).tobytes())
    return h.hexdigest()[:16]


def gather_digests(local: dict) -> dict:
    """All-gather {global_stream: digest} from every rank into one dict (off the hot path)."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return dict(local)
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, local)
    merged = {}
    for d in out:
        merged.update(d)
    return merged
