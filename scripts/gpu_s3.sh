#!/bin/bash
# round-2 session-3 check: GPU tests, critical-stream phases at cfg3, cfg3 bench line (no CPU leg)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q $PYTEST_EXTRA > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
HT_PHASES=1 timeout 600 python scripts/prof_panel.py 3 > gpurun_out/phases3.log 2>&1
tail -3 gpurun_out/phases3.log | cut -c1-600
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --also none $BENCH_EXTRA > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
grep -o '"ms_per_step": [0-9.]*' gpurun_out/bench.log | head -1
