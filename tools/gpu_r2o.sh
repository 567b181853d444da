#!/bin/bash
# static runs of consecutive chunks per CTA: parity, A/B against HEAD, group timing
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_parity_gpu.py tests/test_fuzz_gpu.py tests/test_sequences_gpu.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
for v in base runs base runs; do HFTW_LIBRARY=tools/exp/$v.so python tools/ab_step.py 300; done
for v in base runs; do HFTW_LIBRARY=tools/exp/$v.so python tools/ab_step.py 20; done
timeout 1500 python -m pytest tests/test_group_gpu.py tests/test_dist_gpu.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
timeout 900 python tools/group_one_gpu.py 40 2>&1
