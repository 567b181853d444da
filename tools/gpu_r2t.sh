#!/bin/bash
# decomposed runs on one GPU (groups) with the current defaults, and the un-overlapped
# exchange baseline against the in-kernel pushes
cd $GRAFT_REPO_ROOT
timeout 900 python tools/group_one_gpu.py 40 > gpurun_out/group_one_gpu_r2t.jsonl 2>&1
cat gpurun_out/group_one_gpu_r2t.jsonl
timeout 900 python tools/exchange_baseline.py 20 > gpurun_out/exchange_baseline_r2t.jsonl 2>&1
cat gpurun_out/exchange_baseline_r2t.jsonl
