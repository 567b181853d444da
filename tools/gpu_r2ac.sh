#!/bin/bash
# 10 k-groups as the default: full GPU suite, bench, group timings
cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest_r2ac.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/gputest_r2ac.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_r2ac.json 2>/dev/null; echo "bench rc $?"; head -c 300 gpurun_out/bench_r2ac.json; echo
python tools/ab_step.py 300
timeout 900 python tools/group_one_gpu.py 40 > gpurun_out/group_one_gpu_r2ac.jsonl 2>&1; cat gpurun_out/group_one_gpu_r2ac.jsonl
