# pair kernel: parity first, then a quick timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "pair" 2>&1 | tail -30 | cut -c1-400
timeout 300 python tools/pair_time.py 2>&1 | tail -12
