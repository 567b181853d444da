#!/bin/bash
# full GPU suite + default bench + where a 2x4 rank's pass goes (single domain of the same size)
cd $GRAFT_REPO_ROOT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest_r02r.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/gputest_r02r.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02r.json 2> gpurun_out/bench_r02r.err; echo "bench rc $?"
python tools/ab_step.py 20 auto 790 325 58
python tools/ab_step.py 20 auto 1581 1301 58
head -c 400 gpurun_out/bench_r02r.json
