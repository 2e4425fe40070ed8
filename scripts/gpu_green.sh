#!/bin/bash
# green-partition size x band mode at cfg3 (same box)
mkdir -p gpurun_out
for cfg in "100 sync" "100 conc" "108 conc" "116 conc" "108 sync" "92 conc"; do
  set -- $cfg
  b=""; [ "$2" = sync ] && b="HT_BAND_SYNC=1"
  r=$(env HT_GREEN_SMS=$1 $b timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --also none 2>/dev/null | tail -1 | grep -o '"ms_per_step": [0-9.]*')
  echo "green=$1 band=$2: $r"
done > gpurun_out/green.txt 2>&1
cat gpurun_out/green.txt
