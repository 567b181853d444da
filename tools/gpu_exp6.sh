# A/B of a variant library (tools/exp/$1.so) against tools/exp/head.so: pair parity + timing
V=${1:-unroll2}
mkdir -p gpurun_out
HFTW_LIBRARY=$PWD/tools/exp/$V.so timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "pair or auto" > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log
for i in 1 2; do echo $V; HFTW_LIBRARY=$PWD/tools/exp/$V.so timeout 200 python tools/pair_time.py 2>&1 | grep "kind 1"
  echo head; HFTW_LIBRARY=$PWD/tools/exp/head.so timeout 200 python tools/pair_time.py 2>&1 | grep "kind 1"; done
