#!/bin/bash
# ghost kernel CTA count (tuning build), 2x4 weak ranks: ncu launch times
cd $GRAFT_REPO_ROOT
for n in 74 296 592 1184; do
  HFTW_LIBRARY=tools/exp/tune.so HFTW_GHOST_CTAS=$n timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2ai_$n.csv python tools/group_diag.py 2 4 weak 4 > /dev/null 2>&1
  echo "ctas $n: $(grep pair_ghost gpurun_out/r2ai_$n.csv | awk -F'","' '{print $NF}' | tr -d '"' | sort -n | tr '\n' ' ')"
done
