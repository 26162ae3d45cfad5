"""Per-source-line instructions and stall samples of ONE kernel of an ncu report (files of
the CUDA view matched to the SASS view), with the top stall reasons of the kernel.

    python scripts/ncu_kernel_lines.py REP KERNEL_REGEX [--top 30]
"""
import argparse
import collections
import csv
import io
import subprocess

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("kernel")
ap.add_argument("--top", type=int, default=30)
a = ap.parse_args()
out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", "regex:" + a.kernel], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
heads = [i for i, r in enumerate(rows) if len(r) > 5 and r[0] == "Line No"]
ins, stall, src = collections.Counter(), collections.Counter(), {}
for n, hi in enumerate(heads):
    h = rows[hi]
    fname = rows[hi - 1][1].split("/")[-1] if len(rows[hi - 1]) > 1 else "?"
    iE, iS = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    end = heads[n + 1] - 1 if n + 1 < len(heads) else len(rows)
    cur = None
    for r in rows[hi + 1:end]:
        if len(r) < len(h):
            continue
        if r[0] != "":
            cur = (fname, int(r[0]))
            src[cur] = r[1].strip()[:100]
            continue
        ins[cur] += int(r[iE]) if r[iE].isdigit() else 0
        stall[cur] += int(r[iS]) if r[iS].isdigit() else 0
ti, ts = sum(ins.values()), sum(stall.values())
print(f"{a.kernel}: {ti} warp-instructions, {ts} stall samples")
for k, c in stall.most_common(a.top):
    print(f"{k[0][:16]}:{k[1]:<5d} stall {100 * c / max(ts, 1):5.1f}%  inst {100 * ins[k] / max(ti, 1):5.1f}%  {src.get(k, '')}")
