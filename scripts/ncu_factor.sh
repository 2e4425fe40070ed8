#!/bin/bash
# ncu capture of one window-factorization launch (R3-type single window) at cfg3 shape n=2048,nb=128
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:factor_qr --launch-skip 40 --launch-count 2 \
  -o gpurun_out/factor_ncu -f python scripts/prof_panel.py 3 2048 > gpurun_out/ncu_factor.log 2>&1
ncu -i gpurun_out/factor_ncu.ncu-rep --page details --csv > gpurun_out/factor_details.csv 2>&1
ncu -i gpurun_out/factor_ncu.ncu-rep --page source --csv > gpurun_out/factor_source.csv 2>&1
tail -5 gpurun_out/ncu_factor.log
