#!/bin/bash
# pair unit heights with post-physics storage (tuning build: HFTW_PAIR_CHUNK / _CHUNK2)
cd $GRAFT_REPO_ROOT
for c in "24 12" "28 14" "32 16" "32 8" "24 8" "40 20" "48 24" "32 12" "24 12"; do
  set -- $c
  echo "chunk $1 chunk2 $2: $(HFTW_LIBRARY=tools/exp/tune.so HFTW_PAIR_CHUNK=$1 HFTW_PAIR_CHUNK2=$2 python tools/ab_step.py 300)"
done
