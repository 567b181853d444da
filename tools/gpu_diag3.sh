#!/bin/bash
cd $GRAFT_REPO_ROOT
ncu --set full --clock-control none --import-source on -k regex:step_tma_kernel -s 6 -c 1 -o gpurun_out/prof_tma_dist python tools/group_diag.py 2 1 weak 4 fused_tma > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:step_pair_kernel -s 4 -c 1 -o gpurun_out/prof_pair_dist2 python tools/group_diag.py 2 1 weak 4 > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep | tail -3
