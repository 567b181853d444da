# A/B: pair kernel with one vs two CTA barriers per row; parity first.
mkdir -p gpurun_out
timeout 120 python tools/pair_small.py 100 37 58 > gpurun_out/t0.log 2>&1; echo small=$?
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_output_path.py -x -q > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log
for i in 1 2 3; do echo new; timeout 200 python tools/pair_time.py 2>&1 | grep "kind 1"
  echo bar2; HFTW_LIBRARY=$PWD/tools/exp/bar2.so timeout 200 python tools/pair_time.py 2>&1 | grep "kind 1"; done
