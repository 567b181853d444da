#!/bin/bash
# post-physics storage between the passes of one call: parity, then A/B against HEAD
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_parity_gpu.py tests/test_fuzz_gpu.py tests/test_sequences_gpu.py tests/test_output_path.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
for v in base pform base pform; do HFTW_LIBRARY=tools/exp/$v.so python tools/ab_step.py 300; done
for v in base pform; do HFTW_LIBRARY=tools/exp/$v.so python tools/ab_step.py 20; done
