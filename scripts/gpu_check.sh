#!/bin/bash
# quick GPU check: sanity cases, GPU tests, cfg2 + cfg3 bench detail lines
python scripts/quick.py 2>&1 | tail -12
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for a in "--config 2 --steps 2 --warmup 3" "--steps 1 --warmup 1"; do
  timeout 900 python bench.py $a --no-cpu --no-e2e 2>&1 | python -c "import json,sys; L=sys.stdin.readlines(); d=json.loads(L[-1]) if L and L[-1].startswith('{') else None; print(d['config']['n'], round(d['ms_per_step']), {k:(round(v,4) if isinstance(v,float) else v) for k,v in d['detail'].items()}) if d else print(''.join(L[-5:]))"
done
