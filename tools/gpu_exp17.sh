# single-step TMA kernel: 32-column strips x 8 consumer warps, 2 CTAs/SM (narrow) vs HEAD
mkdir -p gpurun_out
HFTW_LIBRARY=$PWD/tools/exp/narrow.so timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "tma or split or asuca or diffus" > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log
for i in 1 2; do for v in narrow head; do
  HFTW_LIBRARY=$PWD/tools/exp/$v.so HFTW_NO_WAVE=1 timeout 200 python - <<PY
import os, sys, time
sys.path.insert(0, os.getcwd())
from paper_1802_05839_b200 import weather as W
for nx, ny in ((1581, 1301), (256, 256)):
    with W.Context(W.GridConfig(nx=nx, ny=ny, nz=58), kernel="fused_tma") as ctx:
        ctx.init(); ctx.step(20); ctx.sync()
        t0 = time.perf_counter(); ctx.step(200); ctx.sync()
        print("$v", nx, ny, round((time.perf_counter() - t0) * 1e3 / 200, 4), "ms/step")
PY
done; done
