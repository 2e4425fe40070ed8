#!/bin/bash
# env sweep of the cfg3 reduction time: one arm per argument (comma-separated env assignments)
for arm in "" "$@"; do
  printf "%-40s " "${arm:-default}"
  env ${arm//,/ } HT_PHASES=1 timeout 600 python scripts/prof_panel.py ${CFG:-3} 2>&1 | python3 -c "
import sys,re
t=sys.stdin.read()
m=re.search(r\"'seconds': ([0-9.]+)\",t); ph=re.findall(r'critical stream \(s\): (.*?) \|',t)
print(m.group(1) if m else 'FAIL', ph[-1] if ph else t[-300:])"
done
