# split per-row barrier A/B: full pair parity (incl. fuzz/sequences) with the variant, then timing
mkdir -p gpurun_out
export HFTW_LIBRARY=$PWD/tools/exp/splitbar.so
timeout 120 python tools/pair_small.py 100 37 58 > gpurun_out/t0.log 2>&1; echo small=$?
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_fuzz_gpu.py tests/test_sequences_gpu.py tests/test_output_path.py -q -x > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log
unset HFTW_LIBRARY
for i in 1 2; do for v in splitbar head; do echo $v; HFTW_LIBRARY=$PWD/tools/exp/$v.so timeout 200 python tools/pair_time.py 2>&1 | grep "kind 1"; done; done
