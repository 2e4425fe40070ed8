#!/bin/bash
# Round evidence: bench line, ncu captures of the main kernels, cfg2 launch list (outputs in gpurun_out/)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
tail -1 gpurun_out/bench.log | cut -c1-400
bash scripts/ncu_kernel.sh factor_qr_kernel 40 r01_factor_wide 3 4096
bash scripts/ncu_kernel.sh band_wy_kernel 200 r01_band 3 4096
bash scripts/ncu_kernel.sh chain_apply_kernel 300 r01_chain 3 4096
bash scripts/ncu_kernel.sh panel_kernel 10 r01_panel 3 4096
bash scripts/ncu_launches.sh 2
