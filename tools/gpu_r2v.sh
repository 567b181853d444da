#!/bin/bash
cd $GRAFT_REPO_ROOT
HFTW_LIBRARY=tools/exp/sk32.so timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -x -q -p no:cacheprovider -k pair 2>&1 | tail -1
for v in base sk32 base sk32 base sk32; do HFTW_LIBRARY=tools/exp/$v.so python tools/ab_step.py 300; done
