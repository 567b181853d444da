#!/bin/bash
# ghost kernel time without its pushes / waits (tuning build), 2x4 weak and strong
cd $GRAFT_REPO_ROOT
for e in "X=0" "HFTW_DBG_NOPUSH=1" "HFTW_DBG_NOWAIT=1"; do
for sc in weak strong; do
  env HFTW_LIBRARY=tools/exp/tune.so $e timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2ak.csv python tools/group_diag.py 2 4 $sc 4 > /dev/null 2>&1
  echo "$e $sc ghost: $(grep pair_ghost gpurun_out/r2ak.csv | awk -F'","' '{print $NF}' | tr -d '"' | sort -n | awk '{a[NR]=$1} END {print "median", a[int(NR/2)+1], "min", a[1]}')  pair: $(grep step_pair gpurun_out/r2ak.csv | awk -F'","' '{print $NF}' | tr -d '"' | sort -n | awk '{a[NR]=$1} END {print "median", a[int(NR/2)+1]}')"
done; done
