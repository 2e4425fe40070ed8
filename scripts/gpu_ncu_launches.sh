#!/bin/bash
# ncu launch list (per-launch durations, serialized, cold-cache) of ONE cfg3 reduction with the
# current code (HT_PANEL_NOCLUSTER=1: ncu cannot replay cooperative cluster launches).
mkdir -p gpurun_out
python scripts/one_reduction.py 3 0 1 > gpurun_out/one3.log 2>&1 && \
HT_PANEL_NOCLUSTER=1 timeout 3300 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_cfg3.csv python scripts/one_reduction.py 3 0 1 > gpurun_out/ncu_launch.log 2>&1
echo "ncu rc=$?"
python scripts/launch_summary.py gpurun_out/launches_cfg3.csv > gpurun_out/launches_cfg3_summary.txt 2>&1
head -30 gpurun_out/launches_cfg3_summary.txt
