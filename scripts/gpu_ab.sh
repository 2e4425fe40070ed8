#!/bin/bash
# A/B of a development switch on the cfg3 critical stream: $1 = env assignment for the B arm
mkdir -p gpurun_out
timeout 300 python scripts/quick.py 2>&1 | tail -9
for arm in "" "$1"; do
  echo "== arm: ${arm:-default}"
  env $arm HT_PHASES=1 timeout 600 python scripts/prof_panel.py ${CFG:-3} 2>&1 | grep -v "^{" | tail -2
done
