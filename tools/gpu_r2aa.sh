#!/bin/bash
# 9 / 10 k-groups per strip (max 7 / 6 planes per warp) against 8 (max 8)
cd $GRAFT_REPO_ROOT
for v in kg9 kg10; do HFTW_LIBRARY=tools/exp/$v.so timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -x -q -p no:cacheprovider -k "pair or asuca" 2>&1 | tail -1; done
for v in base kg9 kg10 base kg9 kg10; do HFTW_LIBRARY=tools/exp/$v.so python tools/ab_step.py 300; done
for v in base kg9 kg10; do HFTW_LIBRARY=tools/exp/$v.so python tools/ab_step.py 20 auto 790 325 58; done
