"""Per-kernel table of an ncu KLT launch list (gpurun_out/klt_launches_TAG.csv): mean time,
warp-instructions and DRAM reads per launch, one row per kernel.
    python scripts/klt_launch_table.py gpurun_out/klt_launches_TAG.csv"""
import csv
import sys

lines = open(sys.argv[1]).read().splitlines()
start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
rows = list(csv.reader(lines[start:]))
h = rows[0]
ik, im, iv, iid = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = {}
for r in rows[1:]:
    if len(r) < len(h):
        continue
    per.setdefault((int(r[iid]), r[ik].split("(")[0]), {})[r[im]] = float(r[iv].replace(",", ""))
agg = {}
for (i, k), m in per.items():
    a = agg.setdefault(k, [0, 0.0, 0.0, 0.0])
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0.0)
    a[2] += m.get("smsp__inst_executed.sum", 0.0)
    a[3] += m.get("dram__bytes_read.sum", 0.0)
tot = sum(a[1] / a[0] for a in agg.values())
print("| kernel | us per launch | share | warp-instructions | DRAM read |")
print("|---|---|---|---|---|")
for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1] / kv[1][0]):
    t = a[1] / a[0]
    print(f"| {k} | {t:.1f} | {100 * t / tot:.1f} % | {a[2] / a[0] / 1e6:.1f} M | {a[3] / a[0] / 1e6:.1f} MB |")
print(f"| total | {tot:.1f} | | | |")
