#!/bin/bash
# compute-sanitizer passes on small cases: memcheck, racecheck, synccheck, each bounded
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  for cs in "1 256 32" "3 300 128" "4 256 32"; do
    set -- $cs
    timeout 900 $CS --tool $tool --print-limit 20 python scripts/sanitize_case.py $1 $2 $3 > gpurun_out/san_${tool}_cfg$1_$2_$3.log 2>&1
    echo "$tool cfg$1 n=$2 nb=$3 rc=$?: $(tail -3 gpurun_out/san_${tool}_cfg$1_$2_$3.log | tr '\n' ' ')"
  done
done
