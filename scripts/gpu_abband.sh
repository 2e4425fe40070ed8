#!/bin/bash
# A/B: concurrent band (default) vs band on the critical stream (HT_BAND_SYNC=1), same box
mkdir -p gpurun_out
for k in 1 2; do
for v in "" 1; do
  r=$(env ${v:+HT_BAND_SYNC=1} timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --also none 2>/dev/null | tail -1 | grep -o '"ms_per_step": [0-9.]*')
  echo "HT_BAND_SYNC=${v:-unset}: $r"
done
done > gpurun_out/abband.txt 2>&1
cat gpurun_out/abband.txt
