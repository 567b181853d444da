#!/bin/bash
cd $GRAFT_REPO_ROOT
HFTW_LIBRARY=tools/exp/mbu.so timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -x -q -p no:cacheprovider -k "pair or headline" 2>&1 | tail -1
for v in base mbu base mbu base mbu; do HFTW_LIBRARY=tools/exp/$v.so python tools/ab_step.py 300; done
