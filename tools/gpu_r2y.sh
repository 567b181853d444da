#!/bin/bash
# "band" schedule: one unit per CTA, chunk = ny / floor(296 / nstrips), all units in lockstep
cd $GRAFT_REPO_ROOT
for g in "2 4 33" "2 4 8" "2 2 65" "2 2 12" "2 1 131" "2 1 24"; do
  set -- $g
  echo "== $1x$2 strong chunk $3: $(HFTW_LIBRARY=tools/exp/tune.so HFTW_PAIR_CHUNK=$3 HFTW_PAIR_CHUNK2=$3 python tools/group_diag.py $1 $2 strong 20 2>/dev/null | head -2 | tr '\n' ' ')"
done
for c in 261 131 24; do echo "1x1 chunk $c: $(HFTW_LIBRARY=tools/exp/tune.so HFTW_PAIR_CHUNK=$c HFTW_PAIR_CHUNK2=$c python tools/ab_step.py 300)"; done
echo "1x1 chunk 24/12: $(HFTW_LIBRARY=tools/exp/tune.so python tools/ab_step.py 300)"
for c in 33 8; do echo "790x325 single chunk $c: $(HFTW_LIBRARY=tools/exp/tune.so HFTW_PAIR_CHUNK=$c HFTW_PAIR_CHUNK2=$c python tools/ab_step.py 20 auto 790 325 58)"; done
