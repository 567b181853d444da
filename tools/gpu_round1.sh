mkdir -p gpurun_out
set -x
nvidia-smi -L; nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks.mem --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -20
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30
timeout 600 python bench.py --steps 200 --warmup 10 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; tail -5 gpurun_out/bench1.err; cat gpurun_out/bench1.json
timeout 300 python bench.py --steps 50 --warmup 5 --kernel fused_cell --no-e2e --no-cpu-baseline
timeout 300 python bench.py --steps 50 --warmup 5 --kernel split --no-e2e --no-cpu-baseline
timeout 300 python bench.py --steps 50 --warmup 5 --layout kij --no-e2e --no-cpu-baseline
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches1.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_tma -s 3 -c 1 -o gpurun_out/prof1 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu1.log 2>&1; tail -3 gpurun_out/ncu1.log
