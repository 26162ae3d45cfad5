"""Time series of HBM-bound throughput on one GPU: a plain device copy and the C4 DMSGM
step, each run back to back for a few seconds, with NVML memory / GPU temperature, power,
clocks and clock-event reasons sampled alongside.  Question it answers: is the drift of the
per-replay step time within a bench run (52 -> 56 -> 60 us at C4) a property of the kernel
or of the HBM under sustained load (the copy shows the same plateaus)?

  python scripts/hbm_drift.py [--seconds 3] [--cool 5] > gpurun_out/hbm_drift.json
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402


class Nvml:
    def __init__(self):
        import pynvml as nv
        nv.nvmlInit()
        self.nv = nv
        self.h = nv.nvmlDeviceGetHandleByIndex(0)
        self.rows = []
        self._stop = threading.Event()

    def one(self, t0):
        nv, h = self.nv, self.h
        try:
            mt = nv.nvmlDeviceGetFieldValues(h, [nv.NVML_FI_DEV_MEMORY_TEMP])[0]
            mem_temp = mt.value.uiVal if mt.nvmlReturn == 0 else None
        except Exception:
            mem_temp = None
        self.rows.append(dict(
            t=round(time.perf_counter() - t0, 4),
            mem_temp=mem_temp,
            gpu_temp=nv.nvmlDeviceGetTemperature(h, nv.NVML_TEMPERATURE_GPU),
            power_w=nv.nvmlDeviceGetPowerUsage(h) / 1000.0,
            sm_mhz=nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM),
            mem_mhz=nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_MEM),
            reasons=int(nv.nvmlDeviceGetCurrentClocksEventReasons(h)),
        ))

    def run(self, t0, period):
        while not self._stop.is_set():
            self.one(t0)
            time.sleep(period)

    def start(self, t0, period=0.01):
        self._stop.clear()
        self.th = threading.Thread(target=self.run, args=(t0, period), daemon=True)
        self.th.start()

    def stop(self):
        self._stop.set()
        self.th.join()


def timed_series(fn, seconds, chunk, bytes_per_call, stream):
    """Call fn() in chunks of `chunk` calls for ~seconds; GB/s per chunk (CUDA events)."""
    evs = []
    t_end = time.perf_counter() + seconds
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    prev = e0
    n = 0
    while time.perf_counter() < t_end:
        for _ in range(chunk):
            fn()
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        evs.append((prev, e))
        prev = e
        n += 1
        if n % 8 == 0:
            e.synchronize()                  # keep the host at most a few chunks ahead
    torch.cuda.synchronize()
    out = []
    t = 0.0
    for a, b in evs:
        ms = a.elapsed_time(b)
        t += ms
        out.append(dict(t_ms=round(t, 3), us_per_call=round(1000 * ms / chunk, 3),
                        gbs=round(bytes_per_call * chunk / (ms * 1e6), 1)))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=3.0)
    ap.add_argument("--cool", type=float, default=5.0)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    stream = torch.cuda.current_stream()
    nvml = Nvml()
    res = {}

    # 1. plain copy: 8 pairs of 166 MB buffers (332 MB of traffic per call, the C4 step's
    #    algorithmic bytes), rotated so nothing stays in L2
    nb = 165_888_000
    src = [torch.empty(nb, dtype=torch.uint8, device="cuda").fill_(i) for i in range(8)]
    dst = [torch.empty(nb, dtype=torch.uint8, device="cuda") for _ in range(8)]
    k = [0]

    def copy():
        i = k[0] % 8
        dst[i].copy_(src[i])
        k[0] += 1

    for _ in range(20):
        copy()
    time.sleep(args.cool)
    t0 = time.perf_counter()
    nvml.start(t0)
    res["copy"] = timed_series(copy, args.seconds, 40, 2 * nb, stream)
    nvml.stop()
    res["copy_nvml"] = nvml.rows
    nvml.rows = []
    del src, dst
    torch.cuda.empty_cache()

    # 2. the C4 step as bench.py runs it (dmsgm_step_n graph of 40 steps)
    import bench  # noqa: F401  (method_params)
    import paper_1702_05156_b200 as dm
    import synth
    cfg = synth.config("C4ring", S=32)
    ring, Hs = synth.generate_device(cfg, T=8, device="cuda:0")
    frames = ring.repeat(5, 1, 1, 1)
    del ring
    import numpy as np
    Hd = torch.from_numpy(np.ascontiguousarray(np.tile(Hs, (5, 1, 1)))).cuda()
    masks = torch.empty_like(frames)
    ctx = dm.Dmsgm(cfg.W, cfg.H, cfg.N, bench.method_params(dm, 32))
    for i in range(20):
        ctx.step(frames[i], Hd[i], masks[i], stream)
    ctx.step_n(40, frames, Hd, masks, stream)
    torch.cuda.synchronize()
    time.sleep(args.cool)
    t0 = time.perf_counter()
    nvml.start(t0)
    res["c4"] = timed_series(lambda: ctx.step_n(40, frames, Hd, masks, stream), args.seconds, 1,
                             40 * 32 * ctx.info.algorithmic_bytes_per_frame, stream)
    for r in res["c4"]:
        r["us_per_call"] = round(r["us_per_call"] / 40, 3)      # per step
    nvml.stop()
    res["c4_nvml"] = nvml.rows
    ctx.close()
    print(json.dumps(res))


if __name__ == "__main__":
    main()
