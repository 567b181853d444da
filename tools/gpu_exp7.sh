# KIJ lanes-along-k: parity (KIJ paths + fuzz) and timing vs HEAD
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_fuzz_gpu.py tests/test_dist_gpu.py -q -x > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log
for v in new head; do
  if [ $v = head ]; then export HFTW_LIBRARY=$PWD/tools/exp/head.so; else unset HFTW_LIBRARY; fi
  timeout 300 python bench.py --layout kij --kernel fused_tma --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', d['ms_per_step'], d['roofline']['frac'])"
done
