#!/bin/bash
cd $GRAFT_REPO_ROOT
o=gpurun_out/diag7.txt; : > $o
python tools/group_diag.py 2 4 strong 20 >> $o 2>&1
python tools/group_diag.py 2 2 strong 20 >> $o 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,gpc__cycles_elapsed.max --clock-control none --csv --log-file gpurun_out/diag7_launches.csv python tools/group_diag.py 2 4 strong 4 > /dev/null 2>&1
cat $o
