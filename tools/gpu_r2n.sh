#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_sequences_gpu.py tests/test_abi.py -m gpu -x -q -p no:cacheprovider -k "diffus or sequence" 2>&1 | tail -2
for k in 20 100; do python tools/stencil_multi.py $k; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:step_wave -c 3 python tools/stencil_multi.py 20 2>&1 | grep -E "step_wave|duration|bytes" | head -12
