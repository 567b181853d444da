# step_host pipeline: parity tests + the e2e leg of the bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "step_host or reference_api" 2>&1 | tail -5
timeout 300 python -m pytest tests/test_cpp_adapter.py -x -q 2>&1 | tail -3
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_e2e.json 2>gpurun_out/bench_e2e.err; tail -3 gpurun_out/bench_e2e.err
python -c "import json; d=json.load(open('gpurun_out/bench_e2e.json')); print(d['ms_per_step'], json.dumps(d['e2e']))"
