#!/bin/bash
cd $GRAFT_REPO_ROOT
python tools/group_diag.py 2 1 weak 20 > gpurun_out/diag2.txt 2>&1
python tools/group_diag.py 2 1 weak 20 fused_tma >> gpurun_out/diag2.txt 2>&1
python tools/group_diag.py 1 1 weak 20 fused_tma >> gpurun_out/diag2.txt 2>&1
timeout 600 python tools/group_one_gpu.py 40 >> gpurun_out/diag2.txt 2>&1
timeout 900 python -m pytest tests/test_group_gpu.py -q --timeout 600 -p no:cacheprovider -x >> gpurun_out/diag2.txt 2>&1
cat gpurun_out/diag2.txt
