#!/bin/bash
# with the sweep's evict-first hints: is the persisting-L2 window of the panel workspace still worth it?
# (run when the window was still the default and HT_NO_L2PERSIST switched it off; it is now opt-in: HT_L2PERSIST=1)
mkdir -p gpurun_out
out=gpurun_out/persist_ab.txt; : > $out
for v in default nopersist default nopersist; do
  if [ $v = nopersist ]; then export HT_NO_L2PERSIST=1; else unset HT_NO_L2PERSIST; fi
  timeout 600 python bench.py --config 3 --also none --no-e2e --no-cpu --steps 3 --warmup 2 2>/dev/null | \
    python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('$v ms_per_step', d['ms_per_step'], 't_panel', d['detail']['t_panel_s'])" >> $out 2>&1
done
cat $out
