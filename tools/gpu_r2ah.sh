#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pair_ghost -s 4 -c 1 -o gpurun_out/prof_ghost_r2ah python tools/group_diag.py 2 4 weak 4 > /dev/null 2>&1; echo "ncu rc $?"
