#!/bin/bash
cd $GRAFT_REPO_ROOT
python tools/group_diag.py 2 1 weak 20 > gpurun_out/diag4.txt 2>&1
python tools/group_diag.py 2 1 weak 20 fused_tma >> gpurun_out/diag4.txt 2>&1
timeout 600 python tools/group_one_gpu.py 40 >> gpurun_out/diag4.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:step_tma_kernel -s 6 -c 1 -o gpurun_out/prof_tma_dist2 python tools/group_diag.py 2 1 weak 4 fused_tma > /dev/null 2>&1
cat gpurun_out/diag4.txt
