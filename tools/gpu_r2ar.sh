#!/bin/bash
# programmatic dependent launch for the decomposed ghost kernel too
cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests/test_group_gpu.py tests/test_dist_gpu.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -1
for v in base cur base cur; do
  L=tools/exp/base.so; [ $v = cur ] && L=paper_1802_05839_b200/libhftw.so
  echo "$v: $(HFTW_LIBRARY=$L timeout 600 python tools/group_one_gpu.py 40 2x4,2x2,2x1 | tail -3 | python -c 'import sys,json; print([round(json.loads(l)["implied_efficiency"],4) for l in sys.stdin])')"
done
