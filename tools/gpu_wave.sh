mkdir -p gpurun_out
timeout 120 python tools/pair_small.py 100 37 58 >/dev/null 2>&1; echo small_rc=$?
timeout 400 python -m pytest tests/test_parity_gpu.py -x -q -k "multi_step or golden or random_states or hash" 2>&1 | tail -3 | cut -c1-300
for ch in 32 64 128; do HFTW_WAVE_CHUNK=$ch timeout 200 python bench.py --steps 200 --warmup 5 --no-e2e --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('chunk $ch', d['ms_per_step'], d['roofline']['frac'], json.dumps(d['kernels']))"; done
