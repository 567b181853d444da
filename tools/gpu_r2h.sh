#!/bin/bash
# session re-entry sanity: smoke, GPU tests, default bench, pair-kernel ncu with stall reasons
cd $GRAFT_REPO_ROOT
TAG=r02h
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc $?"
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest_$TAG.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/gputest_$TAG.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_pair -s 3 -c 1 -o gpurun_out/prof_pair_$TAG python tools/ab_step.py 20 > /dev/null 2>&1
head -c 700 gpurun_out/bench_$TAG.json
