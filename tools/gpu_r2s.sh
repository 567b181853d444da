#!/bin/bash
# round-2 evidence after post-physics storage / 24-row units: default bench, reference arm,
# stencil line, launch list, pair ncu (inner pass), sanitizers
cd $GRAFT_REPO_ROOT
TAG=${1:-r02s}
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc $?"
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref rc $?"
timeout 900 python bench.py --workload stencil --steps 100 --warmup 5 > gpurun_out/bench_stencil_$TAG.json 2> gpurun_out/bench_stencil_$TAG.err; echo "stencil rc $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline > /dev/null 2>&1; echo "launches rc $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_pair -s 2 -c 1 -o gpurun_out/prof_pair_$TAG python tools/ab_step.py 20 > /dev/null 2>&1; echo "ncu rc $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_wave -s 1 -c 1 -o gpurun_out/prof_wave_stencil_$TAG python tools/stencil_multi.py 20 > /dev/null 2>&1; echo "ncu wave rc $?"
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_small.py > gpurun_out/racecheck_$TAG.log 2>&1
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_small.py > gpurun_out/memcheck_$TAG.log 2>&1
tail -n 2 gpurun_out/racecheck_$TAG.log gpurun_out/memcheck_$TAG.log
