# ASUCA: multi-step launch (wave) vs 200 single-step launches (HFTW_NO_WAVE=1), fused_tma
for nw in 0 1 0 1; do
  HFTW_NO_WAVE=$nw timeout 200 python - <<'PY'
import os, sys, time
sys.path.insert(0, os.getcwd())
from paper_1802_05839_b200 import weather as W
with W.Context(W.GridConfig(nx=1581, ny=1301, nz=58), kernel="fused_tma") as ctx:
    ctx.init(); ctx.step(20); ctx.sync()
    t0 = time.perf_counter(); ctx.step(200); ctx.sync()
    print("NO_WAVE", os.environ["HFTW_NO_WAVE"], (time.perf_counter() - t0) * 1e3 / 200, "ms/step")
PY
done
