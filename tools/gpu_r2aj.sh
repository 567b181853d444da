#!/bin/bash
# ghost kernel with 4 cells per thread and trip (loads before stores): parity, ncu times
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_group_gpu.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -1
for n in 74 148 296; do
  HFTW_LIBRARY=tools/exp/tune.so HFTW_GHOST_CTAS=$n timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2aj_$n.csv python tools/group_diag.py 2 4 weak 4 > /dev/null 2>&1
  echo "weak ctas $n: $(grep pair_ghost gpurun_out/r2aj_$n.csv | awk -F'","' '{print $NF}' | tr -d '"' | sort -n | tr '\n' ' ')"
done
HFTW_LIBRARY=tools/exp/tune.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2aj_s.csv python tools/group_diag.py 2 4 strong 4 > /dev/null 2>&1
echo "strong: $(grep pair_ghost gpurun_out/r2aj_s.csv | awk -F'","' '{print $NF}' | tr -d '"' | sort -n | tr '\n' ' ')"
timeout 600 python tools/group_one_gpu.py 40 2x4
