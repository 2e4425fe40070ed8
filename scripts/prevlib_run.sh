#!/bin/bash
# run irtrace with the previous commit's library (development A/B check)
cp prevlib/lib_prev.so paper_1710_08538_b200/lib/libht_b200.so
REPS=3 python scripts/irtrace.py 3 > gpurun_out/ir_prev.log 2>&1
