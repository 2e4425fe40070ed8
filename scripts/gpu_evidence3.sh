#!/bin/bash
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
tail -1 gpurun_out/bench.log | cut -c1-300
bash scripts/ncu_kernel.sh band_wy_kernel 200 r01_band2 3 4096
bash scripts/ncu_kernel.sh chain_apply_kernel 300 r01_chain2 3 4096
