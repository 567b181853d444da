# parity (pair + full GPU parity) and A/B timing of the working tree vs HEAD
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_output_path.py -x -q > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log
for i in 1 2; do echo new; timeout 200 python tools/pair_time.py 2>&1 | grep "kind 1"
  echo head; HFTW_LIBRARY=$PWD/tools/exp/head.so timeout 200 python tools/pair_time.py 2>&1 | grep "kind 1"; done
