#!/bin/bash
# panel phase profile with and without the sweep's evict-first hints, then the GPU tests
mkdir -p gpurun_out
for m in -1 0; do
  echo "HT_SWEEP_RES_MB=$m" >> gpurun_out/prof_sweep_hints.txt
  HT_SWEEP_RES_MB=$m timeout 600 python scripts/prof_panel.py 3 2>&1 | grep "ht profile" >> gpurun_out/prof_sweep_hints.txt
done
cat gpurun_out/prof_sweep_hints.txt | cut -c1-700
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_s4_hints.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_s4_hints.log
tail -3 gpurun_out/pytest_gpu_s4_hints.log
