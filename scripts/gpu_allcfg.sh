#!/bin/bash
# bench line (cfg3 headline) + one line per config (no CPU/e2e legs) into gpurun_out/
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
for c in 1 2 4 5; do timeout 900 python bench.py --config $c --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_cfg$c.log 2>&1; done
