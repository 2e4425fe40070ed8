#!/bin/bash
# development check: headline-path parity tests + critical-stream phases at cfg3
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu.py -q -x -k "headline or solve_paths or small_sweep or forced or config4_singular or deterministic" 2>&1 | tail -3
HT_PHASES=1 HT_PROFILE=1 timeout 600 python scripts/prof_panel.py ${CFG:-3} 2>&1 | grep "profile\|phases" | tail -2
