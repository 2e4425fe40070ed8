#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/pytest_gpu.log 2>&1
HT_PANEL_NOCLUSTER=1 python -m pytest tests/test_gpu.py -x -q -k "parity or config" > gpurun_out/pytest_nocl.log 2>&1
export HT_PANEL_NOCLUSTER=1
bash scripts/ncu_kernel.sh panel_kernel 10 r01_panel 3 4096
bash scripts/ncu_launches.sh 2
