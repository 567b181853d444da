#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_parity_gpu.py tests/test_group_gpu.py -m gpu -x -q -p no:cacheprovider -k "reverse" 2>&1 | tail -2
python tools/ab_step.py 300
