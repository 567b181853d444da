#!/bin/bash
# small domains: pair passes vs the multi-step single-step launch (wave)
cd $GRAFT_REPO_ROOT
for sz in "790 325 58" "790 650 58" "395 325 58"; do
  python tools/ab_step.py 20 auto $sz
  python tools/ab_step.py 20 fused_tma $sz
done
python tools/group_diag.py 2 4 strong 20 fused_tma 2>/dev/null | head -2
python tools/group_diag.py 2 4 strong 20 2>/dev/null | head -2
