#!/bin/bash
# extra fuzz seeds (random grids x kernels x layouts, random call sequences) after the
# round-2 kernel changes
cd $GRAFT_REPO_ROOT
for seed in 7 99 2026; do
  HFTW_FUZZ_SEED=$seed timeout 1500 python -m pytest tests/test_fuzz_gpu.py tests/test_sequences_gpu.py -m gpu -q -p no:cacheprovider 2>&1 | tail -1
done
