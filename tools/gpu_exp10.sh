# multi-step launch vs single-step launches on the per-rank subdomain sizes
for nw in 0 1; do
  HFTW_NO_WAVE=$nw timeout 300 python - <<'PY'
import os, sys, time
sys.path.insert(0, os.getcwd())
from paper_1802_05839_b200 import weather as W
for nx, ny in ((1581, 1301), (791, 1301), (791, 651), (791, 326)):
    with W.Context(W.GridConfig(nx=nx, ny=ny, nz=58), kernel="fused_tma") as ctx:
        ctx.init(); ctx.step(20); ctx.sync()
        t0 = time.perf_counter(); ctx.step(200); ctx.sync()
        print("NO_WAVE", os.environ["HFTW_NO_WAVE"], nx, ny, round((time.perf_counter() - t0) * 1e3 / 200, 4), "ms/step", flush=True)
PY
done
