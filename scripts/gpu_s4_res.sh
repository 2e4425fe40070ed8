#!/bin/bash
# fused sweep: L2-resident item budget (HT_SWEEP_RES_MB; < 0 = no cache hints)
mkdir -p gpurun_out
out=gpurun_out/sweep_res_cfg${CFG:-3}.txt; : > $out
for m in ${MBS:--1 40 60 80 100 -1 80}; do
  HT_SWEEP_RES_MB=$m timeout 600 python bench.py --config ${CFG:-3} --also none --no-e2e --no-cpu --steps ${ST:-3} --warmup ${WU:-2} 2>/dev/null | \
    python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('res_mb=$m ms_per_step', d['ms_per_step'], 't_panel', d['detail']['t_panel_s'])" >> $out 2>&1
done
cat $out
