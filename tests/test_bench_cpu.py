"""bench.py contract checks that need no GPU: the reference arm (the oracle, this tier's
`--impl reference`) prints one JSON line with the required keys, the warm-up bound is
enforced, and the roofline helpers read the committed profiles/ evidence."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "3"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "dtype", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0 and line["unit"] == "frames/s"
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    assert line["config"]["workload"] == "C4"
    # the same config object as the GPU arm's line (profiles/R2f_bench_C4.json, same defaults)
    with open(os.path.join(ROOT, "profiles", "R2f_bench_C4.json")) as f:
        assert line["config"] == json.loads(f.read())["config"]
    assert 1 <= line["cpu_baseline"]["streams_per_step"] <= line["config"]["streams_per_gpu"]


def test_warmup_bound():
    r = subprocess.run([sys.executable, "bench.py", "--steps", "1", "--warmup", "2"], cwd=ROOT,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode != 0 and "warmup" in r.stderr


def test_roofline_helpers_read_committed_evidence():
    import bench
    peak, src = bench.measured_peak()
    assert peak > 1000 and src
    assert bench.ncu_traffic("C4") and bench.ncu_traffic("C5")
    c4 = bench.ncu_instructions("warp_C4")
    assert c4 and c4 > 1e7
    # a workload without its own capture: the C4 count scaled by the pixel count
    assert abs(bench.ncu_instructions("warp_C4p", pixels=4 * 1920 * 1080) - c4 * 4 / 32) < 1.0
    assert bench.ncu_instructions("warp_C4p") is None


def test_work_roofline_reports_hbm_and_minimal_instructions():
    """The filter / warp kernels are reported against HBM (2 B/px) and against the issue
    time of their minimal instruction count, not against executed
    instructions: a faster kernel raises both fractions, a kernel executing more
    instructions for the same time raises neither."""
    import bench
    assert bench.prefilter_min_instr_per_px(2, 1) == 5 + 1.5 + 1 + 7
    assert bench.prefilter_min_instr_per_px(0, 1) == 7
    assert bench.prefilter_min_instr_per_px(1, 0) == 3 + 2.5
    px = 32 * 1920 * 1080
    r = bench.work_roofline("k", 0.080, px, 14.5, 2 * 14.5 * px / 32, 148, 1965.0, 6454.3, 2.0 * px, None, 0.6, "x")
    assert r["bound"] == "hbm" and abs(r["achieved"] - 2.0 * px / 80e-6 / 1e9) < 1e-6
    assert abs(r["frac"] - r["achieved"] / 6454.3) < 1e-12
    w = r["work"]
    assert abs(w["instr_efficiency"] - 0.5) < 1e-12
    assert abs(w["achieved"] - 14.5 * px / 32 / 80e-6 / 1e9) < 1e-6
    r2 = bench.work_roofline("k", 0.080, px, 14.5, 4 * 14.5 * px / 32, 148, 1965.0, 6454.3, 2.0 * px, None, 0.6, "x")
    assert r2["work"]["frac"] == w["frac"] and r2["frac"] == r["frac"]
