#!/bin/bash
# 16-warp (512-thread) vs 8-warp window factorization: micro-benchmark, parity, cfg3 phases
mkdir -p gpurun_out
cd scripts/micro
for v in "" 1; do
  for a in "256 128 0 0" "256 128 1 0" "256 128 1 128"; do
    echo "HT_FACTOR512=$v $a: $(HT_FACTOR512=$v timeout 60 ./factor_bench ${a%% *} $(echo $a | cut -d' ' -f2) 20 $(echo $a | cut -d' ' -f3) $(echo $a | cut -d' ' -f4) 2>&1 | grep -E 'best|check' | tr '\n' ' ')"
  done
done > ../../gpurun_out/f512_bench.txt 2>&1
cd ../..
cat gpurun_out/f512_bench.txt | cut -c1-300
HT_FACTOR512=1 timeout 900 python -m pytest tests -m gpu -x -q -k "headline or small_sweep or shapes or singular or windows or forced or saddle or general" > gpurun_out/pytest_f512.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_f512.log
tail -2 gpurun_out/pytest_f512.log
HT_FACTOR512=1 HT_PHASES=1 timeout 600 python scripts/prof_panel.py 3 > gpurun_out/phases3_f512.log 2>&1
tail -2 gpurun_out/phases3_f512.log | cut -c1-400
