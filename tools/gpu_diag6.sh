#!/bin/bash
cd $GRAFT_REPO_ROOT
o=gpurun_out/diag6.txt; : > $o
echo "== nopushcode + NOPUSH NOWAIT" >> $o
HFTW_DBG_NOPUSH=1 HFTW_DBG_NOWAIT=1 HFTW_LIBRARY=tools/exp/dist_nopushcode.so python tools/group_diag.py 2 1 weak 20 fused_tma >> $o 2>&1
echo "== nopushcode" >> $o
HFTW_LIBRARY=tools/exp/dist_nopushcode.so python tools/group_diag.py 2 1 weak 20 fused_tma >> $o 2>&1
echo "== dist_t NOPUSH NOWAIT" >> $o
HFTW_DBG_NOPUSH=1 HFTW_DBG_NOWAIT=1 HFTW_LIBRARY=tools/exp/dist_t.so python tools/group_diag.py 2 1 weak 20 fused_tma >> $o 2>&1
echo "== 1x2 and 2x1 strong-size-ranks ( = weak ) multistep off" >> $o
HFTW_LIBRARY=tools/exp/dist_t.so python tools/group_diag.py 1 2 weak 20 fused_tma >> $o 2>&1
cat $o
