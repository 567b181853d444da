#!/bin/bash
# 62-column strips (64 intermediate columns = 2 warps per k-group), one CTA per SM
cd $GRAFT_REPO_ROOT
for v in tx62 tx62kg8; do HFTW_LIBRARY=tools/exp/$v.so timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -x -q -p no:cacheprovider -k "pair or asuca" 2>&1 | tail -1; done
for v in base tx62 tx62kg8 base tx62 tx62kg8; do HFTW_LIBRARY=tools/exp/$v.so python tools/ab_step.py 300; done
