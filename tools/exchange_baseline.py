"""In-kernel halo pushes vs the un-overlapped baseline (HFTW_OPT_EXCHANGE = 1: steps
without the halo protocol, then a separate face-copy kernel per rank), single-step
kernel, decompositions run as groups on ONE GPU (ranks in turn).  Prints ms per step
of the whole group and per rank for each mode.  usage: exchange_baseline.py [K]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1802_05839_b200 import weather as W  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 20
for px, py, scaling in ((2, 1, "strong"), (2, 2, "strong"), (2, 4, "strong"), (2, 4, "weak")):
    nx, ny = (1581 * px, 1301 * py) if scaling == "weak" else (1581, 1301)
    cfg = W.GridConfig(nx=nx, ny=ny, nz=58)
    row = {"ranks": f"{px}x{py}", "scaling": scaling}
    with W.Context(cfg, px=px, py=py, devices=[0] * (px * py), kernel="fused_tma") as ctx:
        ctx.set_option("multistep", -1)
        ctx.init()
        st = torch.cuda.ExternalStream(ctx.rank_context(0).stream)
        for mode in (0, 1, 0, 1):
            ctx.set_option("exchange", mode)
            ctx.step(2)
            ctx.sync()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            ctx.step(K)
            b.record(st)
            ctx.sync()
            ms = a.elapsed_time(b) / K
            key = "in_kernel_push" if mode == 0 else "separate_copy_kernel"
            row[key + "_ms_per_step_per_rank"] = min(ms / (px * py),
                                                     row.get(key + "_ms_per_step_per_rank", 1e9))
    print(json.dumps(row))
