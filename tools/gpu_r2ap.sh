#!/bin/bash
# programmatic dependent launch for the single-step TMA kernel
cd $GRAFT_REPO_ROOT
HFTW_LIBRARY=tools/exp/pdl.so timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_sequences_gpu.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -1
for v in nopdl pdl nopdl pdl; do
  echo "$v stencil: $(HFTW_LIBRARY=tools/exp/$v.so python bench.py --workload stencil --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.load(sys.stdin); print(d["ms_per_step"]*1e3, "us/sweep", d["roofline"]["frac"])')"
  HFTW_LIBRARY=tools/exp/$v.so python tools/ab_step.py 300 fused_tma
done
