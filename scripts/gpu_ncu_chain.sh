#!/bin/bash
# ncu --set full captures of chain_apply_kernel: one live launch inside the cfg3 reduction and
# the standalone measurement-hook launch (scripts/chain_hook.py, first shape).  Read back with
# scripts/ncu_summary.py into profiles/.
mkdir -p gpurun_out
NCU="/usr/local/cuda/bin/ncu --set full --clock-control none --import-source on"
timeout 900 $NCU --kernel-name regex:chain_apply --launch-skip 300 --launch-count 1 -o gpurun_out/chain_cfg3_live -f python scripts/one_reduction.py 3 > gpurun_out/ncu_chain_live.log 2>&1; echo "live rc=$?"
timeout 600 $NCU --kernel-name regex:chain_apply --launch-skip 1 --launch-count 1 -o gpurun_out/chain_cfg3_standalone -f python scripts/chain_hook.py > gpurun_out/ncu_chain_st.log 2>&1; echo "standalone rc=$?"
ls -la gpurun_out/*.ncu-rep
