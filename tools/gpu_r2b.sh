#!/bin/bash
cd $GRAFT_REPO_ROOT
out=gpurun_out/ab2.txt; : > $out
for lib in base distpair2 base distpair2; do
  HFTW_LIBRARY=tools/exp/$lib.so timeout 300 python tools/ab_step.py 300 >> $out 2>&1
done
timeout 1500 python -m pytest tests/test_group_gpu.py tests/test_dist_gpu.py tests/test_parity_gpu.py tests/test_cpp_adapter.py -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_r2b.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_r2b.log
tail -25 gpurun_out/pytest_r2b.log
cat $out
