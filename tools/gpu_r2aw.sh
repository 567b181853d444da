#!/bin/bash
# programmatic dependent launch for the physics kernels (BASELINE configs[2])
cd $GRAFT_REPO_ROOT
HFTW_LIBRARY=tools/exp/ppdl.so timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_sequences_gpu.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -1
for v in base ppdl base ppdl; do for lay in ijk kij; do
  m=0; [ $lay = kij ] && m=1
  echo "$v $lay: $(HFTW_LIBRARY=tools/exp/$v.so python bench.py --workload physics --layout $lay --physics-mode $m --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"],4), "ms", round(d["roofline"]["frac"],3))')"
done; done
