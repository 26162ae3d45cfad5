"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, element by element.

Bar (BASELINE.json north_star): fp32 means/variances within 1e-4 relative, ages
exactly, masks differing in <= 0.01 % of pixels each within 1e-4 of its threshold.
The design target is bitwise equality (canonical operation order, no FMA; DESIGN.md
§2); tests without the fp64 exp branch assert it.
"""
import os

import numpy as np
import pytest
import yaml

import synth
from gpu_util import compare_masks, compare_state, params_pair, run_gpu, run_oracle

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
IDENT = np.eye(3).reshape(9)


@pytest.fixture(params=["default", "generic", "generic_bpt1", "generic_bpt4"])
def kernel_path(request, monkeypatch):
    """default: the persistent shared-memory-staged kernel where it applies (N = 4 with
    even Wb, N = 8); generic: force the register-path kernel (DMSGM_KERNEL=generic);
    generic_bpt1 / _bpt4: that kernel with 1 / 4 blocks per thread at N = 4 (32- / 128-bit
    pixel-row loads, the SURVEY §8(d) ablation variants; other N unchanged)."""
    monkeypatch.delenv("DMSGM_GENERIC_BPT", raising=False)
    if request.param.startswith("generic"):
        monkeypatch.setenv("DMSGM_KERNEL", "generic")
        if request.param != "generic":
            monkeypatch.setenv("DMSGM_GENERIC_BPT", request.param[-1])
    else:
        monkeypatch.delenv("DMSGM_KERNEL", raising=False)
    return request.param


def _check_run(dm, oracle_mod, frames, Hs, N, pg, po, init=None, mode="step", bitwise=False,
               snapshot_every=1):
    gm, gs = run_gpu(dm, frames, Hs, N, pg, init, mode=mode, snapshot_every=snapshot_every)
    om, os_ = run_oracle(oracle_mod, frames, Hs, N, po, init, snapshot_every=snapshot_every)
    nbits = 0
    nmask = 0
    for t in sorted(gs):
        nbits += compare_state(gs[t], os_[t], where=f"t={t}")
        nmask += compare_masks(gm[t], om[t], frames[t], (os_[t][:, 0], os_[t][:, 1]), N,
                               po.theta_d, po.var_floor_classify, where=f"t={t}")
    if bitwise:
        assert nbits == 0, f"{nbits} state values not bitwise equal"
        assert nmask == 0 and np.array_equal(gm, om)
    return gm, gs, nbits, nmask


# ---------------------------------------------------------------------------
with open(os.path.join(GOLDEN, "dsgm_hand_worked.yaml")) as f:
    _CASES = yaml.safe_load(f)["cases"]


@pytest.mark.parametrize("case", _CASES, ids=[c["id"] for c in _CASES])
def test_hand_worked_gpu(cuda_lib, oracle_mod, case):
    dm = cuda_lib
    N = case["N"]
    W = max(4, N)
    frame = np.zeros((N, W), np.uint8)
    for x0 in range(0, W, N):
        frame[:, x0:x0 + N] = np.array(case["pixels"], np.uint8)
    Wb = W // N
    st = np.empty((1, 6, 1, Wb), np.float32)
    st[0, 0:3] = np.array(case["A"], np.float32)[:, None, None]
    st[0, 3:6] = np.array(case["C"], np.float32)[:, None, None]
    pg, po = params_pair(dm, oracle_mod, 1, theta_s=case["theta_s"], decay_lambda=0.0)
    gm, gs, _, _ = _check_run(dm, oracle_mod, frame[None, None], IDENT[None, None], N, pg, po, init=st,
                              bitwise=True)
    out = gs[0][0]
    for i in range(3):
        assert abs(out[i, 0, 0] - case["expect_A"][i]) <= 2e-6 * max(1, abs(case["expect_A"][i]))
        assert abs(out[3 + i, 0, 0] - case["expect_C"][i]) <= 2e-6 * max(1, abs(case["expect_C"][i]))
    assert np.all(gm == case["expect_mask"])


# ---------------------------------------------------------------------------
@pytest.mark.parametrize("name,T", [("C1", 10), ("C2", 60), ("C3", 40)])
def test_sequence_parity(cuda_lib, oracle_mod, name, T, kernel_path):
    cfg = synth.config(name, T=T)
    seq = synth.generate(cfg)
    pg, po = params_pair(cuda_lib, oracle_mod, cfg.S)
    _check_run(cuda_lib, oracle_mod, seq.frames, seq.homographies, cfg.N, pg, po)


@pytest.mark.parametrize("name,T", [("C1", 10), ("C2", 30)])
def test_sequence_parity_bitwise_no_decay(cuda_lib, oracle_mod, name, T):
    cfg = synth.config(name, T=T)
    seq = synth.generate(cfg)
    pg, po = params_pair(cuda_lib, oracle_mod, cfg.S, decay_lambda=0.0)
    _check_run(cuda_lib, oracle_mod, seq.frames, seq.homographies, cfg.N, pg, po, bitwise=True)


# ---------------------------------------------------------------------------
# random states + random homographies, ragged tiles, every block size
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("N,W,H,S", [(1, 100, 20, 2), (2, 72, 30, 2), (4, 200, 52, 3), (4, 1000, 36, 1),
                                     (8, 264, 104, 2), (16, 272, 80, 2), (4, 4, 4, 1), (8, 8, 8, 3)])
@pytest.mark.parametrize("variant", ["default", "decay_often", "no_decay", "appendix_rules"])
def test_random_state_parity(cuda_lib, oracle_mod, N, W, H, S, variant, kernel_path):
    rng = np.random.default_rng(1000 * N + W + H + S + len(variant))
    kw = {"default": {}, "decay_often": dict(decay_var_thresh=100.0, decay_lambda=0.01),
          "no_decay": dict(decay_lambda=0.0),
          "appendix_rules": dict(update_rule=1, classify_rule=1)}[variant]
    pg, po = params_pair(cuda_lib, oracle_mod, S, **kw)
    Wb, Hb = W // N, H // N
    init = np.stack([synth.random_state(rng, Hb, Wb) for _ in range(S)])
    T = 4
    # frames: smooth random fields near the model means plus outliers
    frames = np.empty((T, S, H, W), np.uint8)
    for t in range(T):
        for s in range(S):
            mu = np.kron(init[s, 0], np.ones((N, N)))
            noise = rng.normal(0, rng.uniform(0.5, 20), (H, W))
            out = rng.random((H, W)) < 0.1
            fr = np.where(out, rng.integers(0, 256, (H, W)), mu + noise)
            frames[t, s] = np.clip(np.rint(fr), 0, 255).astype(np.uint8)
    Hs = np.empty((T, S, 9))
    for t in range(T):
        for s in range(S):
            Hs[t, s] = synth.random_homography(rng, W, H, shift=1.5 * N * (1 + t), rot_deg=1.0, zoom=0.02,
                                               persp=1e-4 / max(W, H))
    bitwise = variant in ("no_decay", "appendix_rules")
    _check_run(cuda_lib, oracle_mod, frames, Hs, N, pg, po, init=init, bitwise=bitwise)


def test_exposure_parity(cuda_lib, oracle_mod, kernel_path):
    """Large motions, w <= 0 and far-out projections: exposed blocks reset identically."""
    rng = np.random.default_rng(5)
    N, W, H, S = 4, 64, 32, 6
    pg, po = params_pair(cuda_lib, oracle_mod, S)
    init = np.stack([synth.random_state(rng, H // N, W // N) for _ in range(S)])
    frames = rng.integers(0, 256, (2, S, H, W)).astype(np.uint8)
    Hs = np.empty((2, S, 9))
    Hs[:, 0] = [1, 0, 0, 0, 1, 0, 0, 0, -1]          # w < 0 everywhere
    Hs[:, 1] = [1, 0, 40, 0, 1, -20, 0, 0, 1]         # large shift: partly exposed
    Hs[:, 2] = [1, 0, 0, 0, 1, 0, 0.02, 0, -0.5]      # w changes sign inside the frame
    Hs[:, 3] = [1, 0, 1e7, 0, 1, 0, 0, 0, 1]          # far out
    Hs[:, 4] = [1, 0, 0, 0, 1, 0, 1e31, 0, 1]         # w >= 2^100: degenerate scale (R5), sources near 0
    Hs[:, 5] = [1, 0, 0, 0, 1, 0, 1e29, 0, 1]         # w crosses 2^100 inside the frame
    _check_run(cuda_lib, oracle_mod, frames, Hs, N, pg, po, init=init)


# ---------------------------------------------------------------------------
# API paths: step_n (CUDA graph), step_host (pipelined H2D/D2H), batch invariance, reset
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("T", [1, 4, 5])
def test_step_n_equals_oracle(cuda_lib, oracle_mod, T):
    cfg = synth.config("C2", T=T, S=3)
    seq = synth.generate(cfg)
    pg, po = params_pair(cuda_lib, oracle_mod, 3)
    _check_run(cuda_lib, oracle_mod, seq.frames, seq.homographies, cfg.N, pg, po, mode="step_n")


def test_step_host_equals_oracle(cuda_lib, oracle_mod, kernel_path):
    cfg = synth.config("C4", W=320, H=240, T=5, S=11)
    seq = synth.generate(cfg)
    pg, po = params_pair(cuda_lib, oracle_mod, 11)
    _check_run(cuda_lib, oracle_mod, seq.frames, seq.homographies, cfg.N, pg, po, mode="host")


def test_step_host_async_pipelined(cuda_lib, oracle_mod):
    """dmsgm_step_host_async: T steps enqueued back to back (chunks of consecutive steps
    overlap on the pipe streams), one sync at the end; every step's masks and the final
    state equal the oracle's."""
    import torch
    cfg = synth.config("C4", W=320, H=240, T=6, S=11)
    seq = synth.generate(cfg)
    pg, po = params_pair(cuda_lib, oracle_mod, cfg.S)
    T, S, H, W = seq.frames.shape
    ctx = cuda_lib.Dmsgm(W, H, cfg.N, pg)
    hf = [torch.from_numpy(np.ascontiguousarray(seq.frames[t])).pin_memory() for t in range(T)]
    hh = [torch.from_numpy(np.ascontiguousarray(seq.homographies[t])).pin_memory() for t in range(T)]
    hm = [torch.zeros((S, H, W), dtype=torch.uint8).pin_memory() for _ in range(T)]
    for t in range(T):
        ctx.step_host_async(hf[t], hh[t], hm[t])
    torch.cuda.synchronize()
    gst = np.stack([ctx.get_state(s) for s in range(S)])
    ctx.close()
    om, os_ = run_oracle(oracle_mod, seq.frames, seq.homographies, cfg.N, po, snapshot_every=1)
    for t in range(T):
        compare_masks(hm[t].numpy(), om[t], seq.frames[t], (os_[t][:, 0], os_[t][:, 1]), cfg.N, where=f"t={t}")
    compare_state(gst, os_[T - 1], where="final")


def test_batch_invariance(cuda_lib, oracle_mod):
    """A stream's results do not depend on the batch it is processed in (bitwise)."""
    cfg = synth.config("C4", W=256, H=128, T=6, S=6)
    seq = synth.generate(cfg)
    pg, _ = params_pair(cuda_lib, oracle_mod, 6)
    bm, bs = run_gpu(cuda_lib, seq.frames, seq.homographies, 4, pg)
    for s in (0, 3, 5):
        p1, _ = params_pair(cuda_lib, oracle_mod, 1)
        sm, ss = run_gpu(cuda_lib, seq.frames[:, s:s + 1], seq.homographies[:, s:s + 1], 4, p1)
        assert np.array_equal(sm[:, 0], bm[:, s])
        assert np.array_equal(ss[5][0].view(np.uint32), bs[5][s].view(np.uint32))


def test_reset_and_graph_recapture(cuda_lib, oracle_mod):
    import torch
    dm = cuda_lib
    cfg = synth.config("C2", T=6, S=2)
    seq = synth.generate(cfg)
    pg, po = params_pair(dm, oracle_mod, 2)
    W, H = cfg.W, cfg.H
    ctx = dm.Dmsgm(W, H, 4, pg)
    o = oracle_mod.Oracle(W, H, 4, po)
    f = torch.from_numpy(seq.frames).cuda()
    h = torch.from_numpy(seq.homographies).cuda()
    m = torch.zeros_like(f)
    assert not ctx.is_initialised(0)
    ctx.step_n(3, f[:3], h[:3], m[:3])
    for t in range(3):
        om = o.step(seq.frames[t], seq.homographies[t])
    assert ctx.is_initialised(1)
    ctx.reset(1)
    o.reset(1)
    assert not ctx.is_initialised(1) and ctx.is_initialised(0)
    ctx.step_n(3, f[3:], h[3:], m[3:])
    for t in range(3, 6):
        om = o.step(seq.frames[t], seq.homographies[t])
    torch.cuda.synchronize()
    assert np.array_equal(m[5].cpu().numpy(), om)
    for s in range(2):
        compare_state(ctx.get_state(s)[None], o.get_state(s)[None])
    ctx.close()
    o.close()


def test_argument_errors_gpu(cuda_lib):
    import torch
    dm = cuda_lib
    ctx = dm.Dmsgm(64, 48, 4, dm.Params(num_streams=1))
    f = torch.zeros((1, 48, 64), dtype=torch.uint8, device="cuda")
    h = torch.zeros((1, 9), dtype=torch.float64, device="cuda")
    m = torch.zeros_like(f)
    wide = torch.zeros((1, 48, 80), dtype=torch.uint8, device="cuda")
    with pytest.raises(dm.DmsgmError) as ei:
        ctx.step(wide[:, :, 1:65], h, m)   # misaligned base pointer (the C ABI's check)
    assert ei.value.code == dm.DMSGM_EINVAL
    # the binding's marshalling checks: dtype, shape, device, outer strides
    with pytest.raises(ValueError, match="dtype"):
        ctx.step(f, h.float(), m)          # f32 homographies
    with pytest.raises(ValueError, match="shape"):
        ctx.step(f[:, :, 1:], h, m)
    with pytest.raises(ValueError, match="CUDA"):
        ctx.step(f.cpu(), h, m)
    two = torch.zeros((2, 48, 64), dtype=torch.uint8, device="cuda")
    ctx2 = dm.Dmsgm(64, 48, 4, dm.Params(num_streams=2))
    with pytest.raises(ValueError, match="stride"):
        ctx2.step(torch.zeros((48, 2, 64), dtype=torch.uint8, device="cuda").transpose(0, 1), h.repeat(2, 1), two)
    with pytest.raises(ValueError, match="host"):
        ctx2.step_host(two, h.repeat(2, 1).cpu(), two.cpu())
    ctx2.close()
    bad = np.zeros((6, 12, 16), np.float32)
    bad[0, 0, 0] = np.nan
    with pytest.raises(dm.DmsgmError):
        ctx.set_state(0, bad)
    with pytest.raises(dm.DmsgmError) as ei:
        ctx.get_state(3)
    assert ei.value.code == dm.DMSGM_ESTATE
    ctx.close()


@pytest.mark.slow
@pytest.mark.parametrize("name,T,extra", [("C2", 300, {}), ("C3", 300, {}), ("C2", 300, dict(decay_lambda=0.0)),
                                          ("C2", 300, dict(decay_var_thresh=100.0, decay_lambda=0.01))])
def test_long_sequence_parity(cuda_lib, oracle_mod, name, T, extra):
    """The paper-scale sequences at full length (C2: 300 frames, the paper's 320x240; C3:
    300 of its 1000 frames) through the staged kernel, every 25th state and mask against
    the oracle (the north_star tolerance): long enough for ages to saturate at the cap,
    swaps, resets and the decay's exp branch (R18; frequent in the last case) to recur many
    times -- every state snapshot and all 300 masks bitwise equal (measured: 0 differing
    values in every case, scripts/bitwise_check.py)."""
    cfg = synth.config(name, T=T)
    seq = synth.generate(cfg)
    pg, po = params_pair(cuda_lib, oracle_mod, cfg.S, **extra)
    _check_run(cuda_lib, oracle_mod, seq.frames, seq.homographies, cfg.N, pg, po, bitwise=True,
               snapshot_every=25)
