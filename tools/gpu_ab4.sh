#!/bin/bash
cd $GRAFT_REPO_ROOT
out=gpurun_out/ab4.txt; : > $out
for lib in late early late early late early; do
  HFTW_LIBRARY=tools/exp/$lib.so timeout 300 python tools/ab_step.py 300 >> $out 2>&1
done
timeout 900 python -m pytest tests/test_parity_gpu.py -q --timeout 600 -p no:cacheprovider -k "pair or asuca" >> $out 2>&1
cat $out
