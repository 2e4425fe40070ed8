#!/bin/bash
# round-2 GPU check: all -m gpu tests (no -x; the full-size golden gate deselected until the
# sample file exists), then the bench with every config.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -rA $PYTEST_EXTRA > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -15 gpurun_out/pytest_gpu.log
timeout 1200 python bench.py --steps 3 --warmup 2 $BENCH_EXTRA > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
tail -c 6000 gpurun_out/bench.log
