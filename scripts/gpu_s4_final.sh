#!/bin/bash
# session-4 final evidence: GPU tests, smoke(), the driver-style bench line with the final code
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_s4_final.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_s4_final.log
tail -3 gpurun_out/pytest_gpu_s4_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_s4_final.log 2>&1; tail -1 gpurun_out/smoke_s4_final.log
timeout 1500 python bench.py > gpurun_out/bench_s4_final.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_s4_final.log
tail -c 300 gpurun_out/bench_s4_final.log
