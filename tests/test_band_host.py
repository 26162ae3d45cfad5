"""Row-band split: host logic on CPU, no GPU.

- the band partition;
- dmsgm_band_halo_needed (library host code, the kernel's S1 projection) against the
  oracle's own S1 (dmsgm_oracle_mix_weights) over every block of every band;
- the NCCL-baseline halo exchange in a world-size-3 gloo group: after the exchange each
  rank's halo rows hold exactly its neighbours' own rows.
"""
import os
import socket

import numpy as np
import pytest

import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def band_mod():
    from paper_1702_05156_b200 import build
    build.build()
    from paper_1702_05156_b200 import band, dmsgm
    return band, dmsgm


def test_band_rows(band_mod):
    band, _ = band_mod
    bs = band.band_rows(270, 8)                        # 4K at N = 8
    assert [b.rows for b in bs] == [34] * 6 + [33] * 2
    for Hb in (1, 7, 60, 270):
        for G in range(1, min(Hb, 9) + 1):
            bs = band.band_rows(Hb, G)
            assert bs[0].row0 == 0 and bs[-1].row1 == Hb
            assert all(a.row1 == b.row0 for a, b in zip(bs, bs[1:]))
            assert max(b.rows for b in bs) - min(b.rows for b in bs) <= 1
            assert not bs[0].has_up and not bs[-1].has_down
    with pytest.raises(ValueError):
        band.band_rows(3, 4)


@pytest.mark.parametrize("N", [4, 8])
def test_halo_needed_matches_oracle_projection(band_mod, oracle_mod, N):
    band, dm = band_mod
    rng = np.random.default_rng(N)
    W, H = 24 * N, 20 * N
    Wb, Hb = W // N, H // N
    bands = band.band_rows(Hb, 3)
    for trial in range(12):
        h = synth.random_homography(rng, W, H, shift=rng.uniform(0, 3) * N, rot_deg=2.0, zoom=0.05,
                                    persp=1e-4 / max(W, H))
        for b in bands:
            need = 0
            for bj in range(b.row0, b.row1):
                for bi in range(Wb):
                    exposed, src, w, _ = oracle_mod.mix_weights(W, H, N, h, bi, bj)
                    if exposed:
                        continue
                    for (x, y), wk in zip(src, w):
                        if wk > 0:
                            need = max(need, b.row0 - y, y - (b.row1 - 1))
            assert dm.band_halo_needed(W, H, N, h.reshape(1, 9), b.row0, b.rows) == need, (trial, b)


def test_halo_needed_errors(band_mod):
    _, dm = band_mod
    with pytest.raises(dm.DmsgmError):
        dm.band_halo_needed(64, 64, 8, np.eye(3).reshape(1, 9), 6, 3)     # beyond Hb = 8
    assert dm.band_halo_needed(64, 64, 8, np.eye(3).reshape(1, 9), 0, 8) == 0


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _exchange_worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    from paper_1702_05156_b200.band import band_rows, halo_exchange
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    S, Hb, R, halo = 2, 13, 6, 2
    b = band_rows(Hb, world)[rank]
    truth = torch.arange(S * Hb * R, dtype=torch.float32).view(S, Hb, R)
    buf = torch.full((S, Hb, R), float("nan"))
    buf[:, b.row0:b.row1] = truth[:, b.row0:b.row1]
    sent = halo_exchange(buf, b, halo, rank, world)
    lo, hi = max(0, b.row0 - halo), min(Hb, b.row1 + halo)
    ok = torch.equal(buf[:, lo:hi], truth[:, lo:hi])
    outside = torch.isnan(buf[:, :lo]).all() and torch.isnan(buf[:, hi:]).all()
    expect_sent = (int(b.has_up) + int(b.has_down)) * S * halo * R * 4
    with open(os.path.join(out_dir, f"r{rank}"), "w") as f:
        f.write(f"{int(ok)} {int(outside)} {int(sent == expect_sent)}")
    dist.destroy_process_group()


def test_halo_exchange_gloo_three_ranks(tmp_path, band_mod):
    import torch.multiprocessing as mp
    world = 3
    mp.spawn(_exchange_worker, args=(world, _port(), str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        assert open(tmp_path / f"r{r}").read() == "1 1 1", r
