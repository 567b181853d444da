#!/bin/bash
cd $GRAFT_REPO_ROOT
o=gpurun_out/diag5.txt; : > $o
for v in "" "HFTW_DBG_NOPUSH=1" "HFTW_DBG_NOWAIT=1" "HFTW_DBG_NOPUSH=1 HFTW_DBG_NOWAIT=1"; do
  echo "== dist_t $v" >> $o
  env $v HFTW_LIBRARY=tools/exp/dist_t.so python tools/group_diag.py 2 1 weak 20 >> $o 2>&1
  env $v HFTW_LIBRARY=tools/exp/dist_t.so python tools/group_diag.py 2 1 weak 20 fused_tma >> $o 2>&1
done
echo "== 1x1 tma / pair" >> $o
HFTW_LIBRARY=tools/exp/dist_t.so python tools/group_diag.py 1 1 weak 20 fused_tma >> $o 2>&1
HFTW_LIBRARY=tools/exp/dist_t.so python tools/group_diag.py 1 1 weak 20 >> $o 2>&1
cat $o
