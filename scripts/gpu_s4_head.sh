#!/bin/bash
# session-4 head check in a fresh container: GPU tests, smoke(), the driver-style bench line
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_s4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_s4.log
tail -3 gpurun_out/pytest_gpu_s4.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_s4.log 2>&1; tail -1 gpurun_out/smoke_s4.log
timeout 1500 python bench.py > gpurun_out/bench_s4.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_s4.log
tail -c 400 gpurun_out/bench_s4.log
