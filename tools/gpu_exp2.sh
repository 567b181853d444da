mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_parity_gpu.py -x -q -k "hash or energy_u or random" > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log
for v in 0 1; do HFTW_KIJ_PHYS_WARP=$v timeout 200 python bench.py --workload physics --layout kij --physics-mode 1 --steps 100 --warmup 5 --no-e2e --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('warp=$v', d['ms_per_step'], d['roofline']['frac'])"; done
