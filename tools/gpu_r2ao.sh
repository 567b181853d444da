#!/bin/bash
# final row's j-1 neighbours from registers (one shared load fewer per cell)
cd $GRAFT_REPO_ROOT
HFTW_LIBRARY=tools/exp/bmreg.so timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -x -q -p no:cacheprovider -k "pair or asuca" 2>&1 | tail -1
for v in base bmreg base bmreg base bmreg; do HFTW_LIBRARY=tools/exp/$v.so python tools/ab_step.py 300; done
for v in base bmreg; do HFTW_LIBRARY=tools/exp/$v.so python tools/ab_step.py 20 auto 790 325 58; done
