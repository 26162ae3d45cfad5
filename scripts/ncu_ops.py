"""Executed SASS opcode histogram of the first kernel in an ncu report, per unit of work.
    python scripts/ncu_ops.py REP [--units 4147200] [--top 50]"""
import argparse, collections, csv, io, subprocess
ap = argparse.ArgumentParser(); ap.add_argument("rep"); ap.add_argument("--units", type=float, default=4147200)
ap.add_argument("--top", type=int, default=50); a = ap.parse_args()
out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out))); h = rows[1]
iS, iE, iT = h.index("Source"), h.index("Instructions Executed"), h.index("Thread Instructions Executed")
ops = collections.Counter(); tt = 0
for r in rows[2:]:
    if len(r) < len(h) or not r[iS].split():
        continue
    t = r[iS].split(); op = t[1] if t[0].startswith("@") else t[0]
    if not r[iT].isdigit():
        continue
    ops[op] += int(r[iT]); tt += int(r[iT])
print(f"thread instructions per unit: {tt / a.units:.1f}")
for op, n in ops.most_common(a.top):
    print(f"{op:32s} {n / a.units:7.2f}")
