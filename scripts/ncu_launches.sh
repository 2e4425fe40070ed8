#!/bin/bash
# Launch list (per-kernel device time) of one bench step: ncu --metrics gpu__time_duration.sum
mkdir -p gpurun_out
CFG=${1:-2}
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 40000 --csv \
  --log-file gpurun_out/launches_cfg${CFG}.csv python bench.py --config $CFG --steps 1 --warmup 0 --no-cpu --no-e2e \
  > gpurun_out/ncu_launches_cfg${CFG}.log 2>&1
python scripts/launch_summary.py gpurun_out/launches_cfg${CFG}.csv > gpurun_out/launch_summary_cfg${CFG}.txt
tail -30 gpurun_out/launch_summary_cfg${CFG}.txt
