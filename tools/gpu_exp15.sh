# KIJ conflict-free flat row mapping: KIJ parity with the variant, then full-step KIJ timing
mkdir -p gpurun_out
export HFTW_LIBRARY=$PWD/tools/exp/kijflat.so
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_fuzz_gpu.py tests/test_sequences_gpu.py tests/test_dist_gpu.py -q -x -k "kij or fuzz or sequence or decomposed or physics or golden or hash" > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log
unset HFTW_LIBRARY
for i in 1 2; do for v in kijflat head; do
  HFTW_LIBRARY=$PWD/tools/exp/$v.so timeout 300 python bench.py --layout kij --kernel fused_tma --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],4), round(d['roofline']['frac'],3))"
done; done
