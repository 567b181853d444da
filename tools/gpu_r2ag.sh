#!/bin/bash
# where a weak-scaled rank's pass goes: pair kernel vs ghost kernel per rank (2x4 weak), ncu launch times
cd $GRAFT_REPO_ROOT
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2ag_launches.csv python tools/group_diag.py 2 4 weak 4 > /dev/null 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/r2ag_launches.csv')))
hi=[i for i,r in enumerate(rows) if 'Kernel Name' in r][0]
h=rows[hi]; ki=h.index('Kernel Name'); vi=h.index('Metric Value'); ui=h.index('Metric Unit')
from collections import defaultdict
t=defaultdict(list)
for r in rows[hi+1:]:
    if len(r)<=vi: continue
    t[r[ki].split('(')[0]].append((float(r[vi].replace(',','')), r[ui]))
for k,v in t.items(): print(k[:60], len(v), 'median', sorted(x for x,_ in v)[len(v)//2], v[0][1])
PY
python tools/ab_step.py 20 auto 1581 1301 58
