"""Decomposed runs on the real device path: px x py processes, each with its
own CUDA context and subdomain, halos pushed by the step kernels through CUDA
IPC mappings and ordered by the step flags (include/hftw.h).  Only one GPU is
available in the test harness, so all ranks share cuda:0 (time-sliced
contexts); the protocol is identical across GPUs.  Bitwise vs the oracle.
"""
import os
import socket

import numpy as np
import pytest

import oracle as O
from paper_1802_05839_b200 import weather as W

pytestmark = pytest.mark.gpu


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, shape, grid, steps, layout, kernel, random_init, q, options=None,
            calls=None):
    import torch.distributed as dist
    from paper_1802_05839_b200.dist import DistSimulation
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nx, ny, nz = shape
        cfg = W.GridConfig(nx=nx, ny=ny, nz=nz, diffusion_velocity=0.125,
                           radiation_intensity=0.37, transfer_velocity=0.013)
        sim = DistSimulation(cfg, grid[0], grid[1], layout=layout, device=0, kernel=kernel)
        for name, value in (options or {}).items():
            sim.ctx.set_option(name, value)
        g = O.grid_from(cfg)
        if random_init:
            rng = np.random.default_rng(7)
            n3, n2 = O.shapes(g)
            s0 = O.State(rng.uniform(150, 350, n3), rng.uniform(150, 350, n3),
                         rng.uniform(150, 350, n2), rng.uniform(150, 350, n2))
            st = W.SimState.allocate(cfg)
            for name, arr in st.named().items():
                arr.data[:] = s0.fields()[name]
            sim.upload_state(st)
        else:
            s0 = O.COracle().init(g)
            sim.init()
        if calls is None:
            half = steps // 2
            calls = [half, steps - half]
        assert sum(calls) == steps
        for n in calls:
            sim.step(n)
        sim.sync()
        st = sim.gather_state(0)
        if rank == 0:
            want = O.COracle().steps(g, s0, steps).fields()
            bad = {n: int(np.sum(a.data != want[n])) for n, a in st.named().items()}
            q.put(bad)
        sim.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("shape,grid,steps,layout,kernel,random_init", [
    ((150, 70, 58), (2, 1), 5, "ijk", "auto", False),
    ((150, 70, 58), (1, 2), 4, "ijk", "auto", True),
    ((131, 97, 12), (2, 2), 6, "ijk", "auto", True),
    ((66, 41, 9), (2, 2), 3, "kij", "auto", True),
    ((66, 41, 9), (2, 2), 3, "ijk", "fused_cell", False),
    ((130, 45, 7), (4, 2), 3, "ijk", "auto", True),
    # multi-step launches with in-kernel pushes and per-step flags, many steps per call
    ((131, 97, 12), (2, 2), 11, "ijk", "fused_tma", True),
    ((200, 140, 20), (2, 4), 9, "ijk", "auto", True),
    # two-step passes per rank across processes (CUDA IPC: faces, corners, P')
    ((130, 100, 58), (2, 4), 7, "ijk", "auto", True),
    ((97, 95, 57), (3, 3), 6, "ijk", "auto", False),
])
def test_decomposed_gpu_bitwise(shape, grid, steps, layout, kernel, random_init):
    _run_decomposed(shape, grid, steps, layout, kernel, random_init)


@pytest.mark.parametrize("shape,grid,calls,options", [
    # one launch per step for every call (what a large rank uses), mixed call lengths
    ((131, 97, 12), (2, 2), [1, 3, 1, 2], {"multistep": -1}),
    ((150, 70, 58), (1, 2), [2, 1, 4], {"multistep": -1}),
    # odd process grids (uneven partitions, a rank between two others in both directions)
    ((97, 61, 13), (3, 1), [2, 3], {}),
    ((61, 97, 13), (1, 3), [1, 4], {}),
    ((100, 70, 9), (3, 2), [3, 2], {}),
    # single steps and multi-step launches interleaved on the same step flags
    ((131, 97, 12), (2, 2), [1, 4, 1, 3, 2], {}),
    ((120, 90, 20), (2, 4), [3, 1, 5], {"multistep": 1}),
])
def test_decomposed_call_mix_bitwise(shape, grid, calls, options):
    _run_decomposed(shape, grid, sum(calls), "ijk", "fused_tma", True, options, calls)


def _run_decomposed(shape, grid, steps, layout, kernel, random_init, options=None, calls=None):
    import torch.multiprocessing as mp
    world = grid[0] * grid[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, shape, grid, steps, layout, kernel,
                                               random_init, q, options, calls))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    hung = [p for p in procs if p.exitcode is None]
    for p in hung:
        p.kill()
    assert not hung, "decomposed run hung"
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    bad = q.get(timeout=5)
    assert all(v == 0 for v in bad.values()), bad
