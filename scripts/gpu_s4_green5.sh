#!/bin/bash
# cfg5 (n = 16384, nb = 256): side-stream SM partition size (default 120 SMs at n >= 12288)
mkdir -p gpurun_out
out=gpurun_out/green_cfg5.txt; : > $out
for g in 120 108 132 140; do
  HT_GREEN_SMS=$g timeout 600 python bench.py --config 5 --also none --no-e2e --no-cpu --steps 2 --warmup 1 2>/dev/null | \
    python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('green=$g ms_per_step', d['ms_per_step'], 't_panel', d['detail']['t_panel_s'], 'busy', d['roofline'].get('concurrent',{}).get('busy_s'))" >> $out 2>&1
done
cat $out
