#!/bin/bash
# window factorization times for the basic R3/L3 window (2k x k view) and the shapes sec. 3.5.2's
# block-triangular restoration would put on the same critical chain at l = 4, k = 128
cd scripts/micro && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DHT_NO_STEP_PROF -I../../paper_1710_08538_b200/csrc factor_bench.cu -o factor_bench || exit 1
for s in "256 128" "512 384" "512 128"; do
  echo "== view p x q = $s (dense)"; ./factor_bench $s 20 1 0 | grep "best\|check"
done
