mkdir -p gpurun_out
HFTW_LIBRARY=$PWD/tools/exp/kw.so timeout 600 python -m pytest tests/test_parity_gpu.py -x -q -k pair > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log
for i in 1 2; do echo base; timeout 200 python tools/pair_time.py 2>&1 | grep "kind 1"; echo kw; HFTW_LIBRARY=$PWD/tools/exp/kw.so timeout 200 python tools/pair_time.py 2>&1 | grep "kind 1"; done
