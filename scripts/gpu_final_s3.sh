#!/bin/bash
# session-3 final evidence: the driver-style bench line (all configs, CPU baseline, e2e) and the
# cfg3 ncu launch list (serialized, cold cache) with the final code
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python bench.py > gpurun_out/bench_final.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_final.log
tail -c 600 gpurun_out/bench_final.log
python scripts/one_reduction.py 3 0 1 > gpurun_out/one3.log 2>&1 && \
HT_PANEL_NOCLUSTER=1 timeout 2400 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_cfg3.csv python scripts/one_reduction.py 3 0 1 > gpurun_out/ncu_launch.log 2>&1
echo "ncu rc=$?"
python scripts/launch_summary.py gpurun_out/launches_cfg3.csv > gpurun_out/launches_cfg3_summary.txt 2>&1
gzip -f gpurun_out/launches_cfg3.csv
head -24 gpurun_out/launches_cfg3_summary.txt
