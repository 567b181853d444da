run() { echo -n "$* $EXTRA : "; env "$@" timeout 120 python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline $EXTRA | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4f ms  frac %.3f %s' % (d['ms_per_step'], d['roofline']['frac'], d['config']['kernel']))"; }
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_dist_gpu.py tests/test_output_path.py -x -q 2>&1 | tail -3
EXTRA=""
run HFTW_EVICT=1
run HFTW_EVICT=0
run HFTW_EVICT=1 HFTW_CHUNK=16
run HFTW_EVICT=1 HFTW_CHUNK=64
timeout 300 ncu --set full --clock-control none --import-source on -k regex:step_tma -s 3 -c 1 -o gpurun_out/prof_evict python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 120 python tools/measure_machine.py
ls gpurun_out
