#!/bin/bash
# decomposed pair passes with post-physics storage: parity (groups, processes), group timing
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_group_gpu.py tests/test_dist_gpu.py tests/test_parity_gpu.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
timeout 900 python tools/group_one_gpu.py 40 > gpurun_out/group_one_gpu_r2m.jsonl 2>&1
cat gpurun_out/group_one_gpu_r2m.jsonl
