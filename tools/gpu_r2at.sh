#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests/test_parity_gpu.py tests/test_group_gpu.py -m gpu -x -q -p no:cacheprovider -k "pair_kernel_vs_oracle or group" 2>&1 | tail -2
