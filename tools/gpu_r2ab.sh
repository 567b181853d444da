#!/bin/bash
# k-groups per strip: 8 (base) / 10 / 11 / 12 / 14
cd $GRAFT_REPO_ROOT
for v in kg11 kg12 kg14; do HFTW_LIBRARY=tools/exp/$v.so timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -x -q -p no:cacheprovider -k "pair or asuca" 2>&1 | tail -1; done
for v in base kg10 kg11 kg12 kg14 base kg10 kg11 kg12 kg14; do HFTW_LIBRARY=tools/exp/$v.so python tools/ab_step.py 300; done
for v in base kg10 kg11 kg12 kg14; do HFTW_LIBRARY=tools/exp/$v.so python tools/ab_step.py 20 auto 790 325 58; done
