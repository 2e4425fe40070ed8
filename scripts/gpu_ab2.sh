#!/bin/bash
mkdir -p gpurun_out
cd scripts/micro
{
for a in "256 128 0 0" "256 128 1 128"; do
  set -- $a
  echo "8 warps  $a: $(env -u HT_FACTOR512 timeout 60 ./factor_bench $1 $2 20 $3 $4 2>&1 | grep -E 'best' | cut -c1-200)"
  echo "16 warps $a: $(HT_FACTOR512=1 timeout 60 ./factor_bench $1 $2 20 $3 $4 2>&1 | grep -E 'best' | cut -c1-200)"
done
for a in "256 128 128 0" "256 128 128 1"; do timeout 60 ./band_bench $a 2>&1 | tail -2; done
} > ../../gpurun_out/ab2.txt 2>&1
cat ../../gpurun_out/ab2.txt
