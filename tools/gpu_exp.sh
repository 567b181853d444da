run() { echo -n "$* $EXTRA : "; env "$@" timeout 120 python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline $EXTRA | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4f ms  frac %.3f %s' % (d['ms_per_step'], d['roofline']['frac'], d['config']['kernel']))"; }
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q 2>&1 | tail -3
for l in ijk kij; do for m in 0 1; do EXTRA="--workload physics --layout $l --physics-mode $m"; run X=1; done; done
EXTRA="--workload stencil"; run X=1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:step_tma -s 3 -c 1 -o gpurun_out/prof_stencil python bench.py --workload stencil --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_stencil.csv python bench.py --workload stencil --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out
