#!/bin/bash
cd $GRAFT_REPO_ROOT
o=gpurun_out/diag8.txt; : > $o
for ch in 0 8 12 16 24; do
  for c2 in 0 4; do
    echo "== chunk $ch chunk2 $c2" >> $o
    if [ $ch = 0 ]; then E=""; else E="HFTW_PAIR_CHUNK=$ch"; fi
    if [ $c2 != 0 ]; then E="$E HFTW_PAIR_CHUNK2=$c2"; fi
    env $E HFTW_LIBRARY=tools/exp/tune.so python tools/group_diag.py 2 4 strong 20 2>&1 | head -2 >> $o
  done
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/diag8_launches.csv python tools/group_diag.py 2 4 strong 4 > /dev/null 2>&1
grep pair_ghost gpurun_out/diag8_launches.csv | head -4 | cut -c1-200
cat $o
