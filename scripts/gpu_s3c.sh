#!/bin/bash
mkdir -p gpurun_out
cd scripts/micro
for a in "256 128 0 0" "256 128 1 128" "256 128 1 0"; do set -- $a; timeout 60 ./factor_bench $1 $2 20 $3 $4 2>&1 | grep -E 'best|check' | cut -c1-220; done > ../../gpurun_out/factor_cpasync.txt
cd ../..
cat gpurun_out/factor_cpasync.txt
bash scripts/gpu_s3.sh
