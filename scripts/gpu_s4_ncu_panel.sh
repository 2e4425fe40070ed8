#!/bin/bash
# ncu --set full of one mid-run panel launch (the 21st panel of cfg3: s0 = 2560) with the final code
mkdir -p gpurun_out
python scripts/one_reduction.py 3 0 1 > gpurun_out/one3.log 2>&1 || { echo "plain run failed"; tail gpurun_out/one3.log; exit 1; }
HT_PANEL_NOCLUSTER=1 timeout 900 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:panel_kernel \
  --launch-skip 20 --launch-count 1 -o gpurun_out/panel_s4 -f python scripts/one_reduction.py 3 0 1 > gpurun_out/ncu_panel_s4.log 2>&1
echo "panel ncu rc=$?"
/usr/local/cuda/bin/ncu -i gpurun_out/panel_s4.ncu-rep --page raw --csv > gpurun_out/panel_s4_raw.csv 2>/dev/null
python - <<'PY'
import csv
rows = list(csv.reader(open("gpurun_out/panel_s4_raw.csv")))
hdr, units, vals = rows[0], rows[1], rows[2]
want = ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__registers_per_thread",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__t_sector_hit_rate.pct",
        "smsp__pcsamp_warps_issue_stalled_barrier", "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
        "smsp__pcsamp_warps_issue_stalled_membar", "smsp__pcsamp_warps_issue_stalled_wait",
        "smsp__pcsamp_warps_issue_stalled_short_scoreboard", "smsp__pcsamp_warps_issue_stalled_lg_throttle")
with open("gpurun_out/ncu_panel_s4.txt", "w") as f:
    for h, u, v in zip(hdr, units, vals):
        if h in want or h in ("Kernel Name", "ID"):
            f.write(f"{h} | {v} {u}\n")
print(open("gpurun_out/ncu_panel_s4.txt").read())
PY
