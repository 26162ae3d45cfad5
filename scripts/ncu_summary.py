"""Summarise an ncu capture (+ launch list) into profiles/ (tracked evidence).

    python scripts/ncu_summary.py TAG [--workload C4] [--bench gpurun_out/bench_TAG.json]

Reads gpurun_out/prof_TAG.ncu-rep (ncu --set full) and gpurun_out/launches_TAG.csv
(ncu --metrics gpu__time_duration.sum over the bench's timed NVTX range) and writes
profiles/TAG_ncu_summary.md, profiles/TAG_launches.csv and (for the bench's roofline
"traffic" field) profiles/ncu_traffic_<workload>.json.
"""
from __future__ import annotations

import argparse
import collections
import csv
import io
import json
import os
import shutil
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__bytes_read.sum.per_second", "dram__bytes_write.sum.per_second",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__occupancy_limit_registers",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sectors_srcunit_tex_op_read.sum",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "launch__grid_size", "launch__block_size",
]


def ncu_csv(args):
    out = subprocess.run(["ncu", *args], capture_output=True, text=True, check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("tag")
    ap.add_argument("--workload", default="C4")
    ap.add_argument("--bench", default=None)
    ap.add_argument("--scale", type=float, default=1.0,
                    help="multiply DRAM bytes (capture taken on a smaller batch of the same workload)")
    ap.add_argument("--note", default="")
    args = ap.parse_args()
    go = os.path.join(ROOT, "gpurun_out")
    prof = os.path.join(go, f"prof_{args.tag}.ncu-rep")
    prof_dir = os.path.join(ROOT, "profiles")
    os.makedirs(prof_dir, exist_ok=True)
    lines = [f"# ncu summary {args.tag} ({args.workload})", ""]

    rows = ncu_csv(["-i", prof, "--page", "raw", "--csv"])
    hdr, units, data = rows[0], rows[1], rows[2:]
    kname = hdr.index("Kernel Name")
    per_launch = []
    for d in data:
        rec = {"kernel": d[kname]}
        for m in METRICS:
            if m in hdr:
                rec[m] = (d[hdr.index(m)], units[hdr.index(m)])
        per_launch.append(rec)
    lines.append(f"Source: `ncu --set full --clock-control none --import-source on -k regex:dmsgm_step` "
                 f"({len(per_launch)} launches captured; one row per launch).")
    lines.append("")
    lines.append("| metric | unit | " + " | ".join(f"launch {i}" for i in range(len(per_launch))) + " |")
    lines.append("|---|---|" + "---|" * len(per_launch))
    for m in METRICS:
        if m in hdr:
            vals = [r[m][0] for r in per_launch]
            lines.append(f"| {m} | {per_launch[0][m][1]} | " + " | ".join(vals) + " |")
    lines.append("")

    def num(rec, m, scale):
        v, u = rec[m]
        f = float(v.replace(",", ""))
        return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1.0) if scale else f

    dram = [num(r, "dram__bytes_read.sum", True) + num(r, "dram__bytes_write.sum", True) for r in per_launch]
    dram_per_launch = sum(dram) / len(dram) * args.scale
    lines.append(f"DRAM bytes per launch (read + write, mean{', x%g' % args.scale if args.scale != 1 else ''}): "
                 f"**{dram_per_launch / 1e6:.1f} MB** {args.note}")

    # SASS opcode histogram of the first captured launch (dynamic warp instructions)
    srows = ncu_csv(["-i", prof, "--page", "source", "--csv", "--print-source", "sass"])
    sh = srows[1]
    iS, iE = sh.index("Source"), sh.index("Instructions Executed")
    ops, tot = collections.Counter(), 0
    for r in srows[2:]:
        if len(r) < len(sh) or r[0].startswith("Kernel"):
            if tot:
                break
            continue
        toks = r[iS].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") else toks[0]
        n = int(r[iE])
        ops[op.split(".")[0]] += n
        tot += n
    grid = per_launch[0].get("launch__grid_size", ("0", ""))[0]
    lines.append("")
    lines.append(f"Dynamic warp instructions (launch 0): {tot} ; by opcode (top 25):")
    lines.append("")
    lines.append("| opcode | warp instr | share |")
    lines.append("|---|---|---|")
    for op, n in ops.most_common(25):
        lines.append(f"| {op} | {n} | {n / tot * 100:.1f}% |")

    launches = os.path.join(go, f"launches_{args.tag}.csv")
    if os.path.exists(launches):
        shutil.copy(launches, os.path.join(prof_dir, f"{args.tag}_launches.csv"))
        lrows = [r for r in csv.reader(open(launches)) if len(r) > 5]
        lh = lrows[0]
        ki, vi = lh.index("Kernel Name"), lh.index("Metric Value")
        agg = collections.defaultdict(list)
        for r in lrows[1:]:
            try:
                agg[r[ki]].append(float(r[vi]))
            except ValueError:
                pass
        total = sum(sum(v) for v in agg.values())
        lines += ["", "Launch list of the bench's timed region (`ncu --nvtx --nvtx-include timed/ --metrics "
                      "gpu__time_duration.sum`; cold-cache, serialised):", "",
                  "| kernel | launches | mean ns | share of timed region |", "|---|---|---|---|"]
        for k, v in agg.items():
            lines.append(f"| {k} | {len(v)} | {sum(v) / len(v):.0f} | {sum(v) / total * 100:.1f}% |")
    if args.bench and os.path.exists(args.bench):
        txt = open(args.bench).read().strip().splitlines()
        if txt:
            b = json.loads(txt[-1])
            lines += ["", f"bench.py line of the same build: value {b['value']:.0f} {b['unit']}, "
                          f"ms/step {b['ms_per_step']:.4f}, roofline {json.dumps(b.get('roofline'))}"]
    with open(os.path.join(prof_dir, f"{args.tag}_ncu_summary.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    with open(os.path.join(prof_dir, f"ncu_traffic_{args.workload}.json"), "w") as f:
        json.dump({"dram_bytes_per_launch": dram_per_launch, "source": f"profiles/{args.tag}_ncu_summary.md",
                   "tag": args.tag, "scale": args.scale, "note": args.note}, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
