"""Oracle timing on the host cores (SURVEY §8(d) "Oracle timing"): single core (pinned
with sched_setaffinity) on C2, C3 and a C4 subset, and all cores (one oracle step per
stream per thread) on C4.  Prints one JSON line; reported as a baseline, not a target.

    python scripts/oracle_timing.py [--seconds 8]
"""
import argparse
import json
import os
import platform
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402  (test infrastructure: this script is a measurement of it)
import synth  # noqa: E402


def params(S):
    return oracle.OracleParams(theta_s=4.0, theta_d=4.0, var_init=255.0, age_cap=30.0, var_floor_match=0.1,
                               var_floor_classify=0.25, decay_lambda=0.001, decay_var_thresh=2500.0, num_streams=S)


def run(cfg_name, streams, frames, threads, budget_s, **over):
    cfg = synth.config(cfg_name, T=frames, **over)
    seq = synth.generate(cfg, streams=range(streams))
    o = oracle.Oracle(cfg.W, cfg.H, cfg.N, params(streams))
    masks = np.empty((streams, cfg.H, cfg.W), np.uint8)
    ex = ThreadPoolExecutor(max_workers=threads)

    def step(t):
        list(ex.map(lambda s: o.step_stream(s, seq.frames[t, s], seq.homographies[t, s], masks[s]), range(streams)))
        o.commit()

    step(0)                                      # first frame initialises: untimed
    n, t0 = 0, time.perf_counter()
    while n + 1 < frames and time.perf_counter() - t0 < budget_s:
        step(n + 1)
        n += 1
    wall = time.perf_counter() - t0
    ex.shutdown()
    o.close()
    return {"config": cfg_name, "W": cfg.W, "H": cfg.H, "N": cfg.N, "streams": streams, "frames_timed": n,
            "threads": threads, "frames_per_s": streams * n / wall, "wall_s": wall}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=8.0)
    a = ap.parse_args()
    cores = sorted(os.sched_getaffinity(0))
    out = {"host": platform.processor() or platform.machine(), "cores_available": len(cores), "single_core": [],
           "all_cores": None}
    os.sched_setaffinity(0, {cores[0]})         # 1 core (the SURVEY's taskset run)
    out["single_core"].append(run("C2", 1, 300, 1, a.seconds))
    out["single_core"].append(run("C3", 1, 200, 1, a.seconds))
    out["single_core"].append(run("C4", 2, 40, 1, a.seconds))
    os.sched_setaffinity(0, set(cores))
    out["all_cores"] = run("C4", len(cores), 20, len(cores), a.seconds)
    try:
        with open("/proc/cpuinfo") as f:
            out["cpu_model"] = next(l.split(":", 1)[1].strip() for l in f if l.startswith("model name"))
    except Exception:
        pass
    print(json.dumps(out))


if __name__ == "__main__":
    main()
