#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 300 ncu --set full --clock-control none --import-source on -k regex:pair_ghost -s 2 -c 1 -o gpurun_out/prof_ghost python tools/group_diag.py 2 4 strong 4 > /dev/null 2>&1
timeout 600 python tools/group_one_gpu.py 40 > gpurun_out/group_one_gpu_r2b.jsonl 2>&1
cat gpurun_out/group_one_gpu_r2b.jsonl
