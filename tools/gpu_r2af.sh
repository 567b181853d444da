#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests/test_parity_gpu.py tests/test_fuzz_gpu.py tests/test_sequences_gpu.py tests/test_group_gpu.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -1
python tools/stencil_multi.py 100 | tail -1
timeout 900 python bench.py --workload stencil --steps 100 --warmup 5 > gpurun_out/bench_stencil_r2af.json 2>/dev/null; echo "stencil rc $?"
