#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_r2f.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_r2f.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_r2f.json 2> gpurun_out/bench_r2f.err
tail -5 gpurun_out/pytest_r2f.log; head -c 400 gpurun_out/bench_r2f.json
