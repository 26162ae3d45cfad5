"""Print the headline metrics of an ncu capture: python scripts/ncu_brief.py REP [kernel-regex]."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
want = ["Kernel Name", "gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "launch__grid_size", "sm__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
stalls = [c for c in h if c.startswith("smsp__pcsamp_warps_issue_stalled_") and not c.endswith("_not_issued")]
for r in rows[2:]:
    for w in want:
        if w in h:
            print(f"{w:60s} {r[h.index(w)]}")
    st = sorted(((float(r[h.index(c)] or 0), c) for c in stalls), reverse=True)[:10]
    for v, c in st:
        print(f"  {c[len('smsp__pcsamp_warps_issue_stalled_'):]:40s} {v:.0f}")
