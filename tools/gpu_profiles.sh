# Round profiles: launch list of the default bench command, ncu --set full of the
# multi-step (wavefront) launch, the single-step kernel and the pair kernel.
mkdir -p gpurun_out
TAG=${1:-r01b}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1; wc -l gpurun_out/launches_$TAG.csv
timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_wave -c 1 -o gpurun_out/prof_wave_$TAG python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_wave_$TAG.log 2>&1; tail -1 gpurun_out/ncu_wave_$TAG.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_tma -s 3 -c 1 -o gpurun_out/prof_tma_$TAG python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_tma_$TAG.log 2>&1; tail -1 gpurun_out/ncu_tma_$TAG.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_pair -s 2 -c 1 -o gpurun_out/prof_pair_$TAG python tools/pair_time.py > gpurun_out/ncu_pair_$TAG.log 2>&1; tail -1 gpurun_out/ncu_pair_$TAG.log
