#!/bin/bash
# decomposed-run tests only (multi-process and group contexts)
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_dist_gpu.py tests/test_group_gpu.py tests/test_cpp_adapter.py -q --timeout 600 -p no:cacheprovider -x > gpurun_out/pytest_dist.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_dist.log
tail -15 gpurun_out/pytest_dist.log
