#!/bin/bash
# decomposed ranks: pair unit heights with post-physics storage (tuning build)
cd $GRAFT_REPO_ROOT
for g in "2 4 8 4" "2 4 6 3" "2 4 10 5" "2 4 12 6" "2 4 16 8" "2 2 12 6" "2 2 16 8" "2 2 8 4" "2 2 24 12" "2 1 24 12" "2 1 16 8" "2 1 12 6"; do
  set -- $g
  echo "== $1x$2 strong chunk $3 chunk2 $4: $(HFTW_LIBRARY=tools/exp/tune.so HFTW_PAIR_CHUNK=$3 HFTW_PAIR_CHUNK2=$4 python tools/group_diag.py $1 $2 strong 20 | head -2 | tr '\n' ' ')"
done
