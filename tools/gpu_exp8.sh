# wave (multi-step single-step launch) at ASUCA: current vs before the decomposed-wave commit
for v in new prewdist new prewdist; do
  if [ $v = new ]; then unset HFTW_LIBRARY; else export HFTW_LIBRARY=$PWD/tools/exp/$v.so; fi
  HFTW_WAVE_CHUNK=32 timeout 200 python - <<'PY'
import os, sys, time
sys.path.insert(0, os.getcwd())
from paper_1802_05839_b200 import weather as W
with W.Context(W.GridConfig(nx=1581, ny=1301, nz=58), kernel="fused_tma") as ctx:
    ctx.init(); ctx.step(20); ctx.sync()
    t0 = time.perf_counter(); ctx.step(200); ctx.sync()
    print(os.environ.get("HFTW_LIBRARY", "new")[-14:], (time.perf_counter() - t0) * 1e3 / 200, "ms/step")
PY
done
