#!/bin/bash
# fused sweep: evict-first hint on A's loads (HT_SWEEP_CS = 0 off, 1 by working-set size, 2 always)
mkdir -p gpurun_out
out=gpurun_out/sweep_cs.txt; : > $out
for m in 0 1 2 0 1; do
  HT_SWEEP_CS=$m timeout 600 python bench.py --config ${CFG:-3} --also none --no-e2e --no-cpu --steps 3 --warmup 2 2>/dev/null | \
    python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('cs=$m ms_per_step', d['ms_per_step'], 't_panel', d['detail']['t_panel_s'])" >> $out 2>&1
done
cat $out
