"""Decomposed runs measured on ONE GPU: a group context (hftw_create_multi) with
every rank on cuda:0.  Ranks sharing a device run one launch (or pass) after
the other on one stream, each with the whole GPU, so the group's time per step
divided by the rank count is what one rank's GPU spends per step in an N-GPU
run -- minus the NVLink cost of its halo pushes, which the in-kernel push
overlaps with compute.  Strong scaling: the ASUCA grid split px x py; weak: an
ASUCA-sized subdomain per rank.  Prints one JSON line per decomposition with
the per-rank ms/step and the implied efficiency against the 1-GPU run.
usage: group_one_gpu.py [K] [PXxPY,... strong process grids]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1802_05839_b200 import weather as W  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 40


def timed(ctx, k):
    ctx.step(6)
    ctx.sync()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st = torch.cuda.ExternalStream(ctx.rank_context(0).stream if ctx.group_size > 1 else ctx.stream)
    a.record(st)
    ctx.step(k)
    b.record(st)
    ctx.sync()
    return a.elapsed_time(b) / k


CASES = ((1, 1, "-"), (2, 1, "strong"), (2, 2, "strong"), (2, 4, "strong"),
         (2, 1, "weak"), (2, 2, "weak"), (2, 4, "weak"))
if len(sys.argv) > 2:  # other process grids, strong: e.g. 4x2,8x1,1x8
    CASES = ((1, 1, "-"),) + tuple((int(g.split("x")[0]), int(g.split("x")[1]), "strong")
                                   for g in sys.argv[2].split(","))
base = None
for px, py, scaling in CASES:
    n = px * py
    nx, ny = (1581 * px, 1301 * py) if scaling == "weak" else (1581, 1301)
    cfg = W.GridConfig(nx=nx, ny=ny, nz=58)
    with W.Context(cfg, px=px, py=py, devices=[0] * n) as ctx:
        ctx.init()
        ms = timed(ctx, K)
        kern = ctx.kernel
    per_rank = ms / n
    if base is None:
        base = ms
    eff = base / per_rank if scaling == "weak" else base / (n * per_rank)
    print(json.dumps({"ranks": f"{px}x{py}", "scaling": scaling, "grid": [nx, ny, 58],
                      "kernel": kern, "group_ms_per_step_one_gpu": ms,
                      "per_rank_ms_per_step": per_rank, "implied_efficiency": eff}))
