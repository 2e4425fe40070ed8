#!/bin/bash
# ncu --set full captures of the top kernels at cfg3 (one launch each) + the DMMA peak probe.
mkdir -p gpurun_out
cd scripts/micro && ./dmma_peak > ../../gpurun_out/dmma_peak.txt 2>&1; cd ../..
cat gpurun_out/dmma_peak.txt
NCU="/usr/local/cuda/bin/ncu --set full --clock-control none --import-source on"
export HT_PANEL_NOCLUSTER=1
timeout 900 $NCU --kernel-name regex:chain_apply --launch-skip 300 --launch-count 1 -o gpurun_out/r02_chain_cfg3 -f python scripts/one_reduction.py 3 > gpurun_out/ncu_chain.log 2>&1; echo "chain rc=$?"
timeout 900 $NCU --kernel-name regex:factor_qr --launch-skip 200 --launch-count 1 -o gpurun_out/r02_factor_cfg3 -f python scripts/one_reduction.py 3 > gpurun_out/ncu_factor.log 2>&1; echo "factor rc=$?"
timeout 1500 $NCU --kernel-name regex:panel_kernel --launch-skip 8 --launch-count 1 -o gpurun_out/r02_panel_cfg3 -f python scripts/one_reduction.py 3 > gpurun_out/ncu_panel.log 2>&1; echo "panel rc=$?"
ls -la gpurun_out/*.ncu-rep
