#!/bin/bash
# ncu of the inner pass (PIN+POUT instantiation) of the default 20-step call
cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_pair -s 4 -c 1 -o gpurun_out/prof_pair_r02l python tools/ab_step.py 20 > /dev/null 2>&1
ls -la gpurun_out/prof_pair_r02l.ncu-rep
