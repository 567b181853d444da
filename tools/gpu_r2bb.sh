#!/bin/bash
# 8 vs 10 k-groups on decomposed runs (one-GPU protocol), same box, interleaved
cd $GRAFT_REPO_ROOT
for v in kg8 kg10 kg8 kg10; do
  echo "$v: $(HFTW_LIBRARY=tools/exp/$v.so timeout 600 python tools/group_one_gpu.py 40 | python -c 'import sys,json; print([(json.loads(l)["ranks"]+json.loads(l)["scaling"][0], round(json.loads(l)["per_rank_ms_per_step"],4), round(json.loads(l)["implied_efficiency"],3)) for l in sys.stdin])')"
done
