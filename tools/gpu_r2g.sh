#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2g_launches.csv python tools/group_diag.py 2 4 strong 4 > /dev/null 2>&1
echo "ghost: $(grep pair_ghost gpurun_out/r2g_launches.csv | head -8 | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ')"
echo "tma/pair: $(grep step_pair gpurun_out/r2g_launches.csv | head -8 | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ')"
timeout 600 python tools/group_one_gpu.py 40 > gpurun_out/group_one_gpu_r2g.jsonl 2>&1
python tools/group_diag.py 2 1 weak 20 fused_tma 2>&1 | head -1
timeout 1500 python -m pytest tests/test_group_gpu.py tests/test_dist_gpu.py -q --timeout 600 -p no:cacheprovider 2>&1 | tail -3
cat gpurun_out/group_one_gpu_r2g.jsonl
