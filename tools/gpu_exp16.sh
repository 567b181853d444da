# step_host pipeline: energy_u D2H one block ahead; block count sweep; vs HEAD
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -q -k "step_host or reference" > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log
for i in 1 2; do
  for nb in 32 41; do HFTW_PIPE_BLOCKS=$nb timeout 300 python bench.py --steps 10 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('new nb=$nb e2e', round(d['e2e']['ms_per_step'],2))"; done
  HFTW_LIBRARY=$PWD/tools/exp/head.so timeout 300 python bench.py --steps 10 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('head e2e', round(d['e2e']['ms_per_step'],2))"
done
