#!/bin/bash
# GPU round check: tests, per-phase panel profile, bench lines (outputs under gpurun_out/)
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python scripts/prof_panel.py 2 > gpurun_out/prof2.log 2>&1
timeout 900 python scripts/prof_panel.py 3 > gpurun_out/prof3.log 2>&1
cat gpurun_out/prof2.log gpurun_out/prof3.log | tail -6
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/bench3.log 2>&1
tail -2 gpurun_out/bench3.log
