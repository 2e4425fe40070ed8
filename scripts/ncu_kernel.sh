#!/bin/bash
# usage: scripts/ncu_kernel.sh <kernel-regex> <launch-skip> <tag> [cfg] [n]
K=$1; SKIP=$2; TAG=$3; CFG=${4:-3}; N=${5:-4096}
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:$K --launch-skip $SKIP --launch-count 1 \
  -o gpurun_out/${TAG} -f python scripts/prof_panel.py $CFG $N > gpurun_out/ncu_${TAG}.log 2>&1
ncu -i gpurun_out/${TAG}.ncu-rep --page details --csv > gpurun_out/${TAG}_details.csv 2>&1
ncu -i gpurun_out/${TAG}.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>&1
tail -2 gpurun_out/ncu_${TAG}.log
