#!/bin/bash
# SURVEY §8(d) design-choice evidence: each variant of the step kernel timed by bench.py
# (C4 and C5, CUDA events) and one ncu launch (DRAM bytes, issue-active, instructions).
# Variants: LIB[:ENV=VAL,...]; run from the repo root under gpurun.
OUT=gpurun_out; mkdir -p $OUT
echo "variant,config,us_per_step,frac,dram_MB,issue_active_pct,warp_inst_M" > $OUT/ablation.csv
for v in "$@"; do
  lib=${v%%:*}; envs=""; [ "$lib" != "$v" ] && envs=$(echo ${v#*:} | tr ',' ' ')
  for cfg in C4 C5; do
    # short timed regions (~11 ms at C4, 23 ms at C5): long runs reach the board power cap and
    # drift, which would confound the comparison
    steps=200; [ "$cfg" = "C5" ] && steps=100
    env DMSGM_LIB_PATH=$lib $envs timeout 300 python bench.py --config $cfg --steps $steps --warmup 20 --no-e2e --no-cpu-baseline > $OUT/abl.json 2>$OUT/abl.err
    env DMSGM_LIB_PATH=$lib $envs timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum --clock-control none --csv -k regex:dmsgm_step -s 8 -c 1 python bench.py --config $cfg --steps 4 --warmup 5 --no-e2e --no-cpu-baseline > $OUT/abl_ncu.csv 2>/dev/null
    python - "$v" "$cfg" <<'PY' >> $OUT/ablation.csv
import csv, json, sys
v, cfg = sys.argv[1], sys.argv[2]
b = json.loads(open("gpurun_out/abl.json").read().strip().splitlines()[-1])
m = {}
rows = list(csv.reader(l for l in open("gpurun_out/abl_ncu.csv") if l.startswith('"')))
h = rows[0] if rows else []
if h:
    ni, ui, vi = h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
    for r in rows[1:]:
        unit, val = r[ui], float(r[vi].replace(",", ""))
        m[r[ni]] = val * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
scale = 1                           # the ncu run captures the whole batch (all streams)
dram = (m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)) * scale / 1e6
print(f"{v},{cfg},{1000*b['ms_per_step']:.1f},{b['roofline']['frac']:.3f},{dram:.0f},{m.get('smsp__issue_active.avg.pct_of_peak_sustained_active', 0):.1f},{m.get('smsp__inst_executed.sum', 0)*scale/1e6:.1f}")
PY
    tail -1 $OUT/ablation.csv
  done
done
