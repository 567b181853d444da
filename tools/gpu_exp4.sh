# A/B: rebalanced k-groups (new) vs HEAD; unit-size sweep on the new build.
mkdir -p gpurun_out
timeout 120 python tools/pair_small.py 100 37 58 > gpurun_out/t0.log 2>&1; echo small=$?
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_output_path.py -x -q > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log
for i in 1 2; do echo new; timeout 200 python tools/pair_time.py 2>&1 | grep "kind 1"
  echo head; HFTW_LIBRARY=$PWD/tools/exp/head.so timeout 200 python tools/pair_time.py 2>&1 | grep "kind 1"; done
for c in 8 12 20 24; do echo chunk $c; HFTW_PAIR_CHUNK=$c timeout 200 python tools/pair_time.py 2>&1 | grep "kind 1"; done
