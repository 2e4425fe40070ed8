#!/bin/bash
# development check with A/B arms: parity subset, then critical-stream phases for default and each arg
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu.py -q -x -k "headline or solve_paths or small_sweep or forced or config4_singular or deterministic or streams" 2>&1 | tail -2
for arm in "" "$@"; do
  echo "== arm: ${arm:-default}"
  env $arm HT_PHASES=1 timeout 600 python scripts/prof_panel.py ${CFG:-3} 2>&1 | grep "phases\|seconds" | tail -2 | cut -c1-330
done
