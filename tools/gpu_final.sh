# Round evidence: default bench line, reference arm, launch list and ncu --set full of the
# dominant kernel of the default bench command.
mkdir -p gpurun_out
TAG=${1:-r01f}
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 600 python bench.py > gpurun_out/bench_default_$TAG.json 2> gpurun_out/bench_default_$TAG.err; head -c 300 gpurun_out/bench_default_$TAG.json; echo
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference_$TAG.json 2>&1; tail -c 300 gpurun_out/bench_reference_$TAG.json; echo
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1; wc -l gpurun_out/launches_$TAG.csv
timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_pair -s 4 -c 1 -o gpurun_out/prof_pair_$TAG python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_pair_$TAG.log 2>&1; tail -1 gpurun_out/ncu_pair_$TAG.log
