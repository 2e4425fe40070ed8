#!/bin/bash
# round-2 session-2 baseline: all -m gpu tests, critical-stream phases at cfg3, bench (all configs)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rf $PYTEST_EXTRA > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -8 gpurun_out/pytest_gpu.log
HT_PHASES=1 timeout 600 python scripts/prof_panel.py 3 > gpurun_out/phases3.log 2>&1
tail -4 gpurun_out/phases3.log
timeout 1500 python bench.py --steps 3 --warmup 3 $BENCH_EXTRA > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
tail -c 3000 gpurun_out/bench.log
