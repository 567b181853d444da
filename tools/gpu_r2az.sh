#!/bin/bash
# unit heights again with 10 k-groups + programmatic dependent launch (tuning build)
cd $GRAFT_REPO_ROOT
for c in "24 12" "20 10" "28 14" "24 8" "32 16" "16 8" "24 12"; do set -- $c
  echo "chunk $1/$2: $(HFTW_LIBRARY=tools/exp/tune.so HFTW_PAIR_CHUNK=$1 HFTW_PAIR_CHUNK2=$2 python tools/ab_step.py 300)"
done
