#!/bin/bash
# window factorization times for the shapes of the nb = 128 and nb = 256 chains
cd scripts/micro && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DHT_NO_STEP_PROF -I../../paper_1710_08538_b200/csrc factor_bench.cu -o factor_bench || exit 1
for s in "$@"; do echo "== $s"; ./factor_bench $s | grep "best"; done
