#!/bin/bash
# cfg3 ncu launch list with the final code.  ncu (rc 9) does not profile through the green-context
# side streams, so this capture uses HT_NO_GREEN=1 (ordinary side streams with capped grids: the
# same kernels and per-launch work, serialized and cold-cache under ncu anyway).
mkdir -p gpurun_out
HT_NO_GREEN=1 python scripts/one_reduction.py 3 0 1 > gpurun_out/one3.log 2>&1 && \
HT_NO_GREEN=1 HT_PANEL_NOCLUSTER=1 timeout 2400 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_cfg3.csv python scripts/one_reduction.py 3 0 1 > gpurun_out/ncu_launch.log 2>&1
echo "ncu rc=$?"
python scripts/launch_summary.py gpurun_out/launches_cfg3.csv > gpurun_out/launches_cfg3_summary.txt 2>&1
gzip -f gpurun_out/launches_cfg3.csv
head -24 gpurun_out/launches_cfg3_summary.txt
for g in 24 40 64; do
  r=$(HT_SB_GRID=$g timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --also none 2>/dev/null | tail -1 | grep -o '"ms_per_step": [0-9.]*')
  echo "HT_SB_GRID=$g: $r"
done > gpurun_out/sbgrid.txt
r=$(timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --also none 2>/dev/null | tail -1 | grep -o '"ms_per_step": [0-9.]*')
echo "HT_SB_GRID=unset: $r" >> gpurun_out/sbgrid.txt
cat gpurun_out/sbgrid.txt
