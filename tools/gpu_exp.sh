run() { echo -n "$* : "; env "$@" timeout 120 python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4f ms  frac %.3f' % (d['ms_per_step'], d['roofline']['frac']))"; }
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_dist_gpu.py -x -q 2>&1 | tail -3
run HFTW_CHUNK=32
run HFTW_NS=5
run HFTW_LIBRARY=tools/libhftw_COPY_ONLY.so
run HFTW_LIBRARY=tools/libhftw_NO_STORE.so
timeout 300 ncu --set full --clock-control none --import-source on -k regex:step_tma -s 3 -c 1 -o gpurun_out/prof_r1e python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out
