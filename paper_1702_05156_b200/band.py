"""Row-band split of one large frame over several GPUs.

Block rows are partitioned contiguously into G bands (`band_rows`).  Each band runs its
own context (`Dmsgm.set_band`) and needs the previous state of `halo` block rows on
each side: only S1-S2 (the warp/mix of the previous models, §2.4) read
neighbouring blocks, S4-S8 use the band's own pixels.  Two exchanges are provided:

- "peer" (the product): the step kernel itself stores its edge rows into the
  neighbour's next-state buffer (peer memory over NVLink / NVSwitch; CUDA IPC between
  processes) and a one-thread sync kernel publishes / waits for "step done" flags --
  no NCCL call, no extra copy kernel on the data path;
- "nccl" (the baseline it is measured against): after each step, `halo_exchange` sends
  the edge rows with torch.distributed point-to-point ops into the neighbours' halo rows.

Both give results bitwise equal to the whole-frame step (tests/test_gpu_band.py).  The
Python here is plumbing only: partitioning, handle exchange, marshalling.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Band:
    index: int
    count: int
    row0: int       # first block row
    rows: int       # block rows

    @property
    def row1(self) -> int:
        return self.row0 + self.rows

    @property
    def has_up(self) -> bool:
        return self.index > 0

    @property
    def has_down(self) -> bool:
        return self.index + 1 < self.count


def band_rows(Hb: int, G: int) -> list[Band]:
    """Contiguous partition of Hb block rows into G bands; the first Hb % G bands get one
    more row (4K at N = 8, G = 8: 34 x 6, 33 x 2 -- SURVEY §8(d) C5b)."""
    if G < 1 or Hb < G:
        raise ValueError(f"cannot split {Hb} block rows into {G} bands")
    base, extra = divmod(Hb, G)
    out, r = [], 0
    for i in range(G):
        n = base + (1 if i < extra else 0)
        out.append(Band(i, G, r, n))
        r += n
    return out


def halo_for(width: int, height: int, block: int, homographies, bands: list[Band], margin: int = 0) -> int:
    """One halo for all bands (they must agree): the largest need over the bands for the
    given host homographies, at least 1 (+ margin)."""
    from .dmsgm import band_halo_needed
    need = max(band_halo_needed(width, height, block, homographies, b.row0, b.rows) for b in bands)
    return max(1, need) + margin


def halo_exchange(buf, band: Band, halo: int, rank: int, world: int, group=None):
    """NCCL/gloo baseline exchange on a state buffer viewed as [S][Hb][row_elems]:
    send the band's first `halo` rows to rank - 1 and its last `halo` rows to rank + 1,
    receive the neighbours' edge rows into this band's halo rows (same global rows, since
    every band keeps the whole-grid layout).  Blocking; returns the bytes sent."""
    import torch
    import torch.distributed as dist
    ops, recvs, sent = [], [], 0
    if band.has_up and rank > 0:
        snd = buf[:, band.row0:band.row0 + halo].contiguous()
        rcv = torch.empty_like(snd)
        ops += [dist.P2POp(dist.isend, snd, rank - 1, group), dist.P2POp(dist.irecv, rcv, rank - 1, group)]
        recvs.append((rcv, band.row0 - halo))
        sent += snd.numel() * snd.element_size()
    if band.has_down and rank + 1 < world:
        snd = buf[:, band.row1 - halo:band.row1].contiguous()
        rcv = torch.empty_like(snd)
        ops += [dist.P2POp(dist.isend, snd, rank + 1, group), dist.P2POp(dist.irecv, rcv, rank + 1, group)]
        recvs.append((rcv, band.row1))
        sent += snd.numel() * snd.element_size()
    if ops:   # one group (ncclGroupStart/End under NCCL): no ordering deadlock between the pairs
        for r in dist.batch_isend_irecv(ops):
            r.wait()
    for rcv, r0 in recvs:
        buf[:, r0:r0 + rcv.shape[1]].copy_(rcv)
    return sent


class _CudaArray:
    """__cuda_array_interface__ over a raw device pointer (no copy, no ownership)."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                         "version": 3, "strides": None}


def state_view(ctx, which: int, device):
    """A torch uint8 view [S][Hb][row_bytes] of one of ctx's state buffers (0/1) --
    for the NCCL baseline exchange (marshalling only)."""
    import torch
    b = ctx.get_buffers()
    S, Hb = ctx.params.num_streams, ctx.info.blocks_y
    raw = torch.as_tensor(_CudaArray(b.state[which], b.stream_bytes * S), device=device)
    return raw.view(S, Hb, b.row_bytes)


class BandGroup:
    """G bands of one frame on ONE device in one process (tests, and the 1-GPU C5b bench):
    neighbours attached by plain device pointers.  `streams=None` runs every band on the
    caller's stream (all steps, then all signals, then all waits); a list of CUDA streams
    runs band i on streams[i] with step + sync each (concurrent bands)."""

    def __init__(self, width: int, height: int, block: int, params, G: int, halo: int, device: int = 0,
                 streams=None):
        from .dmsgm import Dmsgm
        self.width, self.height, self.block = width, height, block
        self.bands = band_rows(height // block, G)
        self.halo = halo
        self.ctxs = []
        for b in self.bands:
            c = Dmsgm(width, height, block, params, device)
            c.set_band(b.row0, b.rows, halo if G > 1 else 0)
            self.ctxs.append(c)
        for i, c in enumerate(self.ctxs):
            if i > 0:
                c.attach_peer(0, self.ctxs[i - 1])
            if i + 1 < G:
                c.attach_peer(1, self.ctxs[i + 1])
        self.streams = streams

    def band_slice(self, b: Band):
        N = self.block
        return slice(b.row0 * N, b.row1 * N)

    def band_views(self, frames, masks):
        """Per-band (frames, masks).  A band's images are [S][rows*N][pitch] with streams
        rows*N*pitch apart, so a whole-frame tensor can be sliced in place only for S = 1;
        otherwise pass lists of per-band tensors."""
        if isinstance(frames, (list, tuple)):
            return list(zip(frames, masks))
        if frames.shape[0] != 1:
            raise ValueError("whole-frame tensors can be split in place for S = 1 only; pass per-band lists")
        return [(frames[:, self.band_slice(b)], masks[:, self.band_slice(b)]) for b in self.bands]

    def step(self, frames, homographies, masks):
        """frames / masks: whole-frame [1][H][pitch] CUDA uint8 tensors, or per-band lists."""
        views = self.band_views(frames, masks)
        if len(self.ctxs) == 1:
            self.ctxs[0].step(views[0][0], homographies, views[0][1],
                              stream=self.streams[0] if self.streams else None)
        elif self.streams is None:
            for c, (f, m) in zip(self.ctxs, views):
                c.step(f, homographies, m)
            for c in self.ctxs:
                c.band_signal()
            for c in self.ctxs:
                c.band_wait()
        else:
            for c, (f, m), st in zip(self.ctxs, views, self.streams):
                c.step(f, homographies, m, stream=st)
                c.band_sync(stream=st)

    def step_n(self, T: int, frames, homographies, masks):
        """Per-band lists of [T][S][rows*N][pitch] tensors: one captured graph per band
        (step + sync per frame), each on its own stream."""
        if len(self.ctxs) == 1:
            self.ctxs[0].step_n(T, frames[0], homographies, masks[0],
                                stream=self.streams[0] if self.streams else None)
            return
        if self.streams is None:
            raise ValueError("step_n over bands needs one CUDA stream per band")
        for c, f, m, st in zip(self.ctxs, frames, masks, self.streams):
            c.step_n(T, f, homographies, m, stream=st)

    def get_state(self, s: int):
        """The whole grid assembled from every band's own rows."""
        import numpy as np
        out = None
        for c, b in zip(self.ctxs, self.bands):
            st = c.get_state(s)
            if out is None:
                out = np.empty_like(st)
            out[:, b.row0:b.row1] = st[:, b.row0:b.row1]
        return out

    def set_state(self, s: int, state):
        for c in self.ctxs:
            c.set_state(s, state)

    def status(self) -> list[int]:
        return [c.get_status() for c in self.ctxs]

    def close(self):
        for c in self.ctxs:
            c.close()
        self.ctxs = []


class BandRank:
    """One band per process (torchrun, one GPU per rank).  exchange="peer": CUDA IPC
    handles of the neighbours' state buffers and flags are swapped through
    torch.distributed (plumbing, once) and the kernels store / signal directly;
    exchange="nccl": no peers attached, `halo_exchange` after every step."""

    def __init__(self, width: int, height: int, block: int, params, rank: int, world: int, halo: int,
                 device: int = 0, exchange: str = "peer", group=None):
        import torch
        import torch.distributed as dist

        from .dmsgm import Dmsgm
        self.rank, self.world, self.halo, self.exchange, self.group = rank, world, halo, exchange, group
        self.band = band_rows(height // block, world)[rank]
        self.block = block
        self.device = torch.device("cuda", device)
        self.ctx = Dmsgm(width, height, block, params, device)
        self.ctx.set_band(self.band.row0, self.band.rows, halo if world > 1 else 0)
        if exchange == "peer" and world > 1:
            handles = [None] * world
            dist.all_gather_object(handles, self.ctx.get_ipc_handles(), group=group)
            if self.band.has_up:
                self.ctx.attach_peer_ipc(0, handles[rank - 1])
            if self.band.has_down:
                self.ctx.attach_peer_ipc(1, handles[rank + 1])
            dist.barrier(group=group)
        elif exchange not in ("peer", "nccl"):
            raise ValueError(exchange)

    def step(self, frames_band, homographies, masks_band, stream=None):
        self.ctx.step(frames_band, homographies, masks_band, stream=stream)
        if self.world == 1:
            return
        if self.exchange == "peer":
            self.ctx.band_sync(stream=stream)
        else:
            nxt = self.ctx.get_buffers().parity      # the buffer the step just wrote
            halo_exchange(state_view(self.ctx, nxt, self.device), self.band, self.halo, self.rank, self.world,
                          group=self.group)

    def step_n(self, T: int, frames_band, homographies, masks_band, stream=None):
        """T frames [T][S][rows*N][pitch].  peer: one CUDA graph (step + sync per frame);
        nccl: T host-driven steps, each followed by the NCCL exchange."""
        if self.exchange == "peer" or self.world == 1:
            self.ctx.step_n(T, frames_band, homographies, masks_band, stream=stream)
        else:
            for t in range(T):
                self.step(frames_band[t], homographies[t], masks_band[t], stream=stream)

    def close(self):
        self.ctx.close()
