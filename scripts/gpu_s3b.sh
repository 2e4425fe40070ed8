#!/bin/bash
mkdir -p gpurun_out
bash scripts/gpu_s3.sh
HT_NO_GREEN=1 timeout 300 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -k regex:inv_diag_kernel -c 3 \
  python scripts/one_reduction.py 3 0 1 > gpurun_out/ncu_invdiag.log 2>&1; echo "ncu rc=$?"
grep -E "inv_diag|gpu__time_duration" gpurun_out/ncu_invdiag.log | head -8
timeout 600 python scripts/side_vs_critical.py 3 > gpurun_out/side_vs_critical.txt 2>&1
cat gpurun_out/side_vs_critical.txt
