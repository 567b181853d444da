#!/bin/bash
# strong scaling of the ASUCA grid over other process grids (group on one GPU)
cd $GRAFT_REPO_ROOT
timeout 900 python tools/group_one_gpu.py 40 2x4,4x2,8x1,1x8,2x2,4x1,1x4,2x1,1x2
