#!/bin/bash
cd $GRAFT_REPO_ROOT
o=gpurun_out/r2d.txt; : > $o
python tools/group_diag.py 2 1 weak 20 >> $o 2>&1
python tools/group_diag.py 2 1 weak 20 fused_tma >> $o 2>&1
python tools/group_diag.py 2 4 weak 20 >> $o 2>&1
timeout 600 python tools/group_one_gpu.py 40 >> $o 2>&1
timeout 600 python tools/ab_step.py 300 >> $o 2>&1
timeout 1500 python -m pytest tests/test_group_gpu.py tests/test_dist_gpu.py tests/test_parity_gpu.py tests/test_cpp_adapter.py -q --timeout 600 -p no:cacheprovider >> $o 2>&1
cat $o
