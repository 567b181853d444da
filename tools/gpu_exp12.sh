# single-step TMA kernel: L2 prefetch distance A/B (HFTW_NO_WAVE irrelevant at ASUCA: one launch per step)
mkdir -p gpurun_out
HFTW_LIBRARY=$PWD/tools/exp/pf8.so timeout 600 python -m pytest tests/test_parity_gpu.py -q -x -k "tma or auto or asuca" > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log
for rep in 1 2; do for v in head pf4 pf8 pf12; do
  HFTW_LIBRARY=$PWD/tools/exp/$v.so timeout 200 python - <<PY
import os, sys, time
sys.path.insert(0, os.getcwd())
from paper_1802_05839_b200 import weather as W
with W.Context(W.GridConfig(nx=1581, ny=1301, nz=58), kernel="fused_tma") as ctx:
    ctx.init(); ctx.step(20); ctx.sync()
    t0 = time.perf_counter(); ctx.step(200); ctx.sync()
    print("$v", round((time.perf_counter() - t0) * 1e3 / 200, 4), "ms/step")
PY
done; done
