"""GPU parity of the row-band split: one frame split into G
block-row bands, each its own context, edge rows stored into the neighbours' buffers by
the step kernel, step-done flags exchanged by the sync kernel.  The assembled result
must equal the whole-frame run -- bitwise against the whole-frame CUDA path (same
arithmetic, only the partition differs) and within the north_star bar against the
oracle (which runs the whole frame, single-threaded).
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import synth
from gpu_util import compare_masks, compare_state, params_pair, run_gpu, run_oracle

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bands(dm, frames, Hs, N, params, G, halo=None, mode="one_stream", init=None):
    """frames u8 [T][S][H][W] -> (masks, states {t: [S][6][Hb][Wb]}, statuses) through BandGroup."""
    import torch

    from paper_1702_05156_b200.band import BandGroup, band_rows, halo_for
    T, S, H, W = frames.shape
    bands = band_rows(H // N, G)
    if halo is None:
        halo = halo_for(W, H, N, Hs.reshape(-1, 9), bands)
    dev = torch.device("cuda", 0)
    streams = None if mode == "one_stream" else [torch.cuda.Stream(dev) for _ in range(G)]
    grp = BandGroup(W, H, N, params, G, halo, streams=streams)
    if init is not None:
        for s in range(S):
            grp.set_state(s, init[s])
    pitch = (W + 15) // 16 * 16
    masks = np.empty_like(frames)
    states = {}
    # per-band device images [T][S][rows*N][pitch]
    fb = [torch.zeros((T, S, b.rows * N, pitch), dtype=torch.uint8, device=dev) for b in bands]
    mb = [torch.zeros_like(f) for f in fb]
    for b, f in zip(bands, fb):
        f[..., :W] = torch.from_numpy(np.ascontiguousarray(frames[:, :, b.row0 * N:b.row1 * N])).to(dev)
    h = torch.from_numpy(np.ascontiguousarray(Hs)).to(dev)
    if mode == "step_n":
        torch.cuda.synchronize()
        grp.step_n(T, fb, h, mb)
        torch.cuda.synchronize()
        states[T - 1] = np.stack([grp.get_state(s) for s in range(S)])
    else:
        for t in range(T):
            if streams is not None:
                for st in streams:
                    st.wait_stream(torch.cuda.current_stream())
            grp.step([f[t] for f in fb], h[t], [m[t] for m in mb])
            torch.cuda.synchronize()
            states[t] = np.stack([grp.get_state(s) for s in range(S)])
    for b, m in zip(bands, mb):
        masks[:, :, b.row0 * N:b.row1 * N] = m[..., :W].cpu().numpy()
    st = grp.status()
    grp.close()
    return masks, states, st


def _check(dm, oracle_mod, frames, Hs, N, pg, po, G, mode="one_stream", init=None, halo=None):
    bm, bs, status = run_bands(dm, frames, Hs, N, pg, G, halo=halo, mode=mode, init=init)
    assert status == [0] * G, status
    snap = 1 if mode != "step_n" else frames.shape[0]
    wm, ws = run_gpu(dm, frames, Hs, N, pg, init, mode="step", snapshot_every=snap)
    om, os_ = run_oracle(oracle_mod, frames, Hs, N, po, init, snapshot_every=snap)
    for t in sorted(bs):
        assert np.array_equal(bs[t].view(np.uint32), ws[t].view(np.uint32)), f"t={t}: band state != whole-frame"
        compare_state(bs[t], os_[t], where=f"t={t}")
    assert np.array_equal(bm, wm), "band masks != whole-frame masks"
    last = max(bs)
    compare_masks(bm[last], om[last], frames[last], (os_[last][:, 0], os_[last][:, 1]), N, po.theta_d,
                  po.var_floor_classify)


@pytest.mark.parametrize("G", [2, 3, 5])
def test_band_sequence_c2(cuda_lib, oracle_mod, G):
    cfg = synth.config("C2", T=25)
    seq = synth.generate(cfg)
    pg, po = params_pair(cuda_lib, oracle_mod, cfg.S)
    _check(cuda_lib, oracle_mod, seq.frames, seq.homographies, cfg.N, pg, po, G)


@pytest.mark.parametrize("mode", ["streams", "step_n"])
def test_band_sequence_n8_concurrent(cuda_lib, oracle_mod, mode):
    """N = 8 (the C5b block size), bands on concurrent streams (sync kernels really wait)."""
    cfg = synth.config("C3", T=16, N=8)
    seq = synth.generate(cfg)
    pg, po = params_pair(cuda_lib, oracle_mod, cfg.S)
    _check(cuda_lib, oracle_mod, seq.frames, seq.homographies, 8, pg, po, 4, mode=mode)


@pytest.mark.parametrize("N,W,H,S,G", [(4, 200, 96, 2, 3), (8, 264, 136, 2, 4), (1, 64, 40, 2, 3),
                                       (2, 72, 48, 1, 2), (16, 272, 160, 2, 3)])
def test_band_random_states(cuda_lib, oracle_mod, N, W, H, S, G, monkeypatch):
    """Random states, vertical motion of up to ~2 blocks (halo from the host helper),
    every block size (N = 1, 2, 16: the register-path kernel), S > 1 streams."""
    rng = np.random.default_rng(77 + N + G)
    pg, po = params_pair(cuda_lib, oracle_mod, S, decay_lambda=0.0)
    Wb, Hb = W // N, H // N
    init = np.stack([synth.random_state(rng, Hb, Wb) for _ in range(S)])
    T = 3
    frames = rng.integers(0, 256, (T, S, H, W)).astype(np.uint8)
    Hs = np.empty((T, S, 9))
    for t in range(T):
        for s in range(S):
            Hs[t, s] = synth.random_homography(rng, W, H, shift=2.0 * N, rot_deg=0.5, zoom=0.01,
                                               persp=1e-5 / max(W, H))
    _check(cuda_lib, oracle_mod, frames, Hs, N, pg, po, G, init=init)


def test_band_generic_kernel(cuda_lib, oracle_mod, monkeypatch):
    monkeypatch.setenv("DMSGM_KERNEL", "generic")
    cfg = synth.config("C2", T=12)
    seq = synth.generate(cfg)
    pg, po = params_pair(cuda_lib, oracle_mod, cfg.S)
    _check(cuda_lib, oracle_mod, seq.frames, seq.homographies, cfg.N, pg, po, 3)


@pytest.mark.parametrize("generic", [False, True])
def test_band_halo_overflow_detected(cuda_lib, oracle_mod, monkeypatch, generic):
    """A vertical shift of 3 blocks with a 1-row halo: the kernel flags it (status bit 0)
    and the next step refuses to run (DMSGM_ESTATE)."""
    import torch

    from paper_1702_05156_b200.band import BandGroup
    if generic:
        monkeypatch.setenv("DMSGM_KERNEL", "generic")
    N, W, H = 8, 128, 128
    pg, _ = params_pair(cuda_lib, oracle_mod, 1)
    grp = BandGroup(W, H, N, pg, 2, 1)
    dev = torch.device("cuda", 0)
    f = torch.randint(0, 256, (1, H, W), dtype=torch.uint8, device=dev)
    m = torch.zeros_like(f)
    h0 = torch.tensor(np.eye(3).reshape(1, 9), device=dev)
    grp.step(f, h0, m)                                  # first frame: no source reads
    h = torch.tensor(np.array([[1, 0, 0, 0, 1, 3.0 * N, 0, 0, 1]], np.float64), device=dev)
    grp.step(f, h, m)
    torch.cuda.synchronize()
    assert cuda_lib.band_halo_needed(W, H, N, h.cpu().numpy(), 0, 8) == 3
    with pytest.raises(cuda_lib.DmsgmError, match="ESTATE"):
        grp.step(f, h, m)
    st = grp.status()
    assert st[0] & 1, st                                 # the upper band reads rows 8..10 of the lower
    grp.close()


def test_band_api_errors(cuda_lib, oracle_mod):
    pg, _ = params_pair(cuda_lib, oracle_mod, 1)
    a = cuda_lib.Dmsgm(64, 64, 8, pg)
    b = cuda_lib.Dmsgm(64, 64, 8, pg)
    with pytest.raises(cuda_lib.DmsgmError):
        a.set_band(4, 5, 1)                              # beyond Hb = 8
    with pytest.raises(cuda_lib.DmsgmError):
        a.attach_peer(1, b)                              # no band set
    a.set_band(0, 4, 1)
    with pytest.raises(cuda_lib.DmsgmError):
        a.attach_peer(0, b)                              # nothing above row 0
    b.set_band(4, 4, 1)
    a.attach_peer(1, b)
    b.attach_peer(0, a)
    assert a.info.kernels_per_step == 2 and a.info.band_rows == 4 and a.info.band_halo == 1
    c = cuda_lib.Dmsgm(64, 32, 8, pg)
    c.set_band(2, 2, 1)
    with pytest.raises(cuda_lib.DmsgmError):
        b.attach_peer(0, c)                              # different grid
    a.set_band(0, 8, 0)                                  # back to whole frame
    assert a.info.kernels_per_step == 1
    for x in (a, b, c):
        x.close()


def test_band_two_processes_ipc(cuda_lib):
    """Two processes on the same GPU, one band each, neighbours attached through CUDA IPC
    (the torchrun path): masks and states equal the whole-frame single-process run."""
    env = dict(os.environ, DMSGM_BAND_TIMEOUT_MS="20000")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "band_ipc_worker.py")], env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "IPC-OK" in r.stdout, r.stdout[-2000:]
