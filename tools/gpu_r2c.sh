#!/bin/bash
cd $GRAFT_REPO_ROOT
out=gpurun_out/ab3.txt; : > $out
for lib in base distpair3 base distpair3; do
  HFTW_LIBRARY=tools/exp/$lib.so timeout 300 python tools/ab_step.py 300 >> $out 2>&1
done
timeout 600 python tools/group_one_gpu.py 40 > gpurun_out/group_one_gpu.jsonl 2>&1
timeout 1500 python -m pytest tests/test_group_gpu.py tests/test_dist_gpu.py -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_r2c.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_r2c.log
tail -5 gpurun_out/pytest_r2c.log
cat $out gpurun_out/group_one_gpu.jsonl
