#!/bin/bash
cd $GRAFT_REPO_ROOT
o=gpurun_out/diag9.txt; : > $o
for cfg in "2 2 strong" "2 1 strong" "1 1 strong"; do
  for ch in 0 8 12 16; do
    if [ $ch = 0 ]; then E=""; else E="HFTW_PAIR_CHUNK=$ch"; fi
    echo "== $cfg chunk $ch" >> $o
    env $E HFTW_LIBRARY=tools/exp/tune.so python tools/group_diag.py $cfg 20 2>&1 | head -1 >> $o
  done
done
for v in "HFTW_GHOST_CTAS=16" "HFTW_GHOST_CTAS=74" "HFTW_GHOST_CTAS=296" "HFTW_DBG_NOWAIT=1"; do
  env $v HFTW_LIBRARY=tools/exp/tune.so timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/diag9_ghost.csv -k regex:pair_ghost -c 4 python tools/group_diag.py 2 4 strong 4 > /dev/null 2>&1
  echo "== ghost $v: $(grep pair_ghost gpurun_out/diag9_ghost.csv | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ')" >> $o
done
cat $o
