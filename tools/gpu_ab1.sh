#!/bin/bash
# A/B: unit prefetch in the pair kernel, and the unit height with it
cd $GRAFT_REPO_ROOT
out=gpurun_out/ab1.txt; : > $out
for lib in base prefetch base prefetch; do
  HFTW_LIBRARY=tools/exp/$lib.so timeout 300 python tools/ab_step.py 300 >> $out 2>&1
done
for ch in 12 16 20 24 32; do
  echo "chunk $ch" >> $out
  HFTW_PAIR_CHUNK=$ch HFTW_LIBRARY=tools/exp/prefetch_t.so timeout 300 python tools/ab_step.py 300 >> $out 2>&1
done
cat $out
