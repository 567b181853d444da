mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_parity_gpu.py -x -q -k "multi_step or golden or hash" 2>&1 | tail -2 | cut -c1-300
for alt in 0 1; do for ch in 32 48 64; do HFTW_WAVE_ALT=$alt HFTW_WAVE_CHUNK=$ch timeout 200 python bench.py --steps 200 --warmup 5 --no-e2e --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('alt $alt chunk $ch', round(d['ms_per_step'],4), round(d['roofline']['frac'],4))"; done; done
