#!/bin/bash
cd $GRAFT_REPO_ROOT
python tools/group_diag.py 2 1 weak 20 > gpurun_out/diag1.txt 2>&1
python tools/group_diag.py 2 1 weak 20 fused_tma >> gpurun_out/diag1.txt 2>&1
python tools/group_diag.py 1 1 weak 20 >> gpurun_out/diag1.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/diag1_launches.csv python tools/group_diag.py 2 1 weak 6 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:step_pair_kernel -s 4 -c 1 -o gpurun_out/prof_pair_dist python tools/group_diag.py 2 1 weak 4 > /dev/null 2>&1
cat gpurun_out/diag1.txt
