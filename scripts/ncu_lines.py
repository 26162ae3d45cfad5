"""Per-CUDA-source-line dynamic instruction and stall breakdown of an ncu report.

    python scripts/ncu_lines.py gpurun_out/prof_TAG.ncu-rep [--top 50] [--units N]
"""
import argparse
import csv
import io
import subprocess

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("--top", type=int, default=50)
ap.add_argument("--units", type=float, default=0, help="divide counts by this (e.g. blocks/32)")
a = ap.parse_args()
out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
agg = {}
fn = "?"
func0 = None
for r in rows:
    if r and r[0] == "File Path":
        fn = r[1].split("/")[-1]
        continue
    if r and r[0] == "Function Name":
        if func0 is None:
            func0 = r[1]
        elif r[1] != func0:
            break
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    iE = hdr.index("Instructions Executed")
    iW = hdr.index("Warp Stall Sampling (All Samples)")
    if r[0] != "-" and r[2] == "-":
        try:
            key = (fn, int(r[0]))
            n, w = int(r[iE]), int(r[iW])
        except ValueError:
            continue
        if n or w:
            agg[key] = (n, w, r[1].strip()[:100])
tot = sum(v[0] for v in agg.values())
totw = sum(v[1] for v in agg.values())
u = a.units or 1.0
print(f"total attributed warp instr {tot} ({tot / u:.1f} per unit), stall samples {totw}")
for (f, l), (n, w, s) in sorted(agg.items(), key=lambda kv: -kv[1][0])[: a.top]:
    print(f"{n / u:8.1f} {100 * w / max(totw, 1):5.1f}% {f[:18]:18s} L{l:<4d} {s}")
