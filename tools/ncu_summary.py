"""One CSV line of headline metrics per kernel launch of an ncu report.

    python tools/ncu_summary.py rep.ncu-rep > summary.csv
"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__inst_executed.sum", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__t_sector_hit_rate.pct",
        "lts__t_sector_hit_rate.pct", "launch__shared_mem_per_block_dynamic",
        "smsp__pcsamp_warps_issue_stalled_wait", "smsp__pcsamp_warps_issue_stalled_short_scoreboard",
        "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
        "smsp__pcsamp_warps_issue_stalled_branch_resolving", "smsp__pcsamp_warps_issue_stalled_selected"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
units = rows[1]
idx = [h.index(k) for k in KEYS if k in h]
w = csv.writer(sys.stdout)
w.writerow(["Kernel Name"] + [h[i] for i in idx])
w.writerow([""] + [units[i] for i in idx])
for r in rows[2:]:
    w.writerow([r[h.index("Kernel Name")]] + [r[i] for i in idx])
