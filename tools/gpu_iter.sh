# usage: bash tools/gpu_iter.sh TAG [extra bench args]
TAG=${1:-it}; shift
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 300 python bench.py --steps 200 --warmup 10 --no-e2e --no-cpu-baseline "$@" | tee gpurun_out/bench_$TAG.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('VALUE', d['value'], 'ms', d['ms_per_step'], 'frac', d['roofline']['frac'], d['clocks'])"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_tma -s 3 -c 1 -o gpurun_out/prof_$TAG python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline "$@" > gpurun_out/ncu_$TAG.log 2>&1; tail -2 gpurun_out/ncu_$TAG.log
