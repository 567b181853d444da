#!/bin/bash
# L2 prefetch of the slab D rows ahead (pair kernel), exchange baseline after the push_box fix
cd $GRAFT_REPO_ROOT
for v in base pf2 pf3 pf5 base pf2 pf3 pf5; do HFTW_LIBRARY=tools/exp/$v.so python tools/ab_step.py 300; done
timeout 900 python -m pytest tests/test_group_gpu.py -m gpu -x -q -p no:cacheprovider -k "exchange" 2>&1 | tail -1
timeout 900 python tools/exchange_baseline.py 20 2>&1
