"""The multi-GPU decomposition plan, checked on CPU with gloo (world size 2..8).

The plan (partition, neighbours, cyclic-partner slots, where each face lands)
comes from the library's host-only hftw_plan_rank -- the same function the
GPU path uses.  Each rank runs a test-local numpy restatement of the fused
kernel's LOCAL semantics on its subdomain (halo slots start as NaN, so any
read of an unfilled slot poisons the result), pushes its faces to the
neighbours over gloo exactly where the plan says, and rank 0 compares the
gathered state with the oracle BITWISE after several steps.
"""
import os
import socket

import numpy as np
import pytest

import oracle as O
from paper_1802_05839_b200 import weather as W

W_, E_, S_, N_ = range(4)


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


# ---------------------------------------------------------------------------
# pure plan properties (no processes)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("shape,grid", [((16, 16, 8), (2, 1)), ((17, 13, 5), (3, 3)),
                                        ((9, 7, 2), (2, 4)), ((1581, 1301, 58), (2, 4)),
                                        ((33, 29, 11), (8, 1)), ((5, 4, 3), (4, 2)),
                                        ((4, 4, 4), (1, 4))])
def test_plan_covers_grid_once_and_faces_agree(shape, grid):
    nx, ny, nz = shape
    px, py = grid
    cfg = W.GridConfig(nx=nx, ny=ny, nz=nz)
    plans = [W.plan(cfg, px, py, r) for r in range(px * py)]
    cover = np.zeros((nx + 2, ny + 2), dtype=int)
    for p in plans:
        i0 = 0 if p["own_w"] else 1
        i1 = p["lnx"] + 1 if p["own_e"] else p["lnx"]
        j0 = 0 if p["own_s"] else 1
        j1 = p["lny"] + 1 if p["own_n"] else p["lny"]
        cover[p["gi0"] + i0:p["gi0"] + i1 + 1, p["gj0"] + j0:p["gj0"] + j1 + 1] += 1
        assert p["lnx"] >= 1 and p["lny"] >= 1
    assert np.all(cover == 1)
    for p in plans:
        for d in range(4):
            q = p["nbr"][d]
            if q < 0:
                continue
            n = plans[q]
            assert n["nbr"][d ^ 1] == p["rank"]          # the relation is symmetric
            if d in (W_, E_):                             # same row of ranks: same j range
                assert (p["face_lo"][d], p["face_hi"][d]) == (n["face_lo"][d ^ 1],
                                                              n["face_hi"][d ^ 1])
                slot = p["send_slot"][d]
                assert slot in (-1, 0, n["lnx"] + 1, n["lnx"] + 2)
            else:
                assert p["lnx"] == n["lnx"]
                assert p["send_slot"][d] in (-1, 0, n["lny"] + 1, n["lny"] + 2)


def test_plan_rejects_too_fine_decomposition():
    with pytest.raises(W.HftwError):
        W.plan(W.GridConfig(nx=3, ny=3, nz=2), 4, 1, 0)


# ---------------------------------------------------------------------------
# numpy restatement of the kernel's local semantics + gloo face exchange
# ---------------------------------------------------------------------------
def phys(E, SF, PB, g):
    P = E + g.radiation_intensity
    P[:, :, 0] = P[:, :, 0] - g.transfer_velocity * (P[:, :, 0] - SF)
    P[:, :, -1] = P[:, :, -1] - g.transfer_velocity * (P[:, :, -1] - PB)
    return P


def local_step(E, SF, PB, p, g):
    """One fused step on a local array indexed [li+1, lj+1, k-1]; returns
    (U over owned cells, NaN elsewhere; post-physics P)."""
    nx, ny, nz = p["lnx"], p["lny"], E.shape[2]
    dv = g.diffusion_velocity
    c2, c5, c6 = 1 - 2.0 * dv, 1 - 5.0 * dv, 1 - 6.0 * dv
    P = phys(E, SF, PB, g)
    U = np.full_like(E, np.nan)
    o = 1  # array offset of local index 0
    I = slice(1 + o, nx + 1 + o)
    J = slice(1 + o, ny + 1 + o)
    Im, Ip = slice(o, nx + o), slice(2 + o, nx + 2 + o)
    Jm, Jp = slice(o, ny + o), slice(2 + o, ny + 2 + o)
    s = P[Im, J] + P[Ip, J]
    s = s + P[I, Jm]
    s = s + P[I, Jp]
    inner = np.empty_like(s)
    if nz > 2:
        t = (s[:, :, 1:-1] + P[I, J, :-2]) + P[I, J, 2:]
        inner[:, :, 1:-1] = c6 * P[I, J, 1:-1] + dv * t
    inner[:, :, 0] = c5 * P[I, J, 0] + dv * (s[:, :, 0] + P[I, J, 1])
    inner[:, :, -1] = c5 * P[I, J, -1] + dv * (s[:, :, -1] + P[I, J, -2])
    U[I, J] = inner
    if p["own_s"]:
        U[I, o] = c2 * P[I, o] + dv * (P[I, p["sfar"] + o] + P[I, 1 + o])
    if p["own_n"]:
        U[I, ny + 1 + o] = c2 * P[I, ny + 1 + o] + dv * (P[I, ny + o] + P[I, p["nfar"] + o])
    j0 = 0 if p["own_s"] else 1
    j1 = ny + 1 if p["own_n"] else ny
    Jo = slice(j0 + o, j1 + 1 + o)
    if p["own_w"]:
        U[o, Jo] = c2 * P[o, Jo] + dv * (P[1 + o, Jo] + P[p["wfar"] + o, Jo])
    if p["own_e"]:
        U[nx + 1 + o, Jo] = c2 * P[nx + 1 + o, Jo] + dv * (P[p["efar"] + o, Jo] + P[nx + o, Jo])
    return U, P


def face(A, p, d):
    """My outgoing face in direction d (values of owned cells)."""
    o = 1
    if d in (W_, E_):
        li = 1 if d == W_ else p["lnx"]
        return A[li + o, p["face_lo"][d] + o:p["face_hi"][d] + 1 + o].copy()
    lj = 1 if d == S_ else p["lny"]
    return A[p["face_lo"][d] + o:p["face_hi"][d] + 1 + o, lj + o].copy()


def put(A, q, d, slot, vals):
    """Write neighbour q's face (it sent in direction d) into my slot."""
    o = 1
    if d in (W_, E_):
        A[slot + o, q["face_lo"][d] + o:q["face_hi"][d] + 1 + o] = vals
    else:
        A[q["face_lo"][d] + o:q["face_hi"][d] + 1 + o, slot + o] = vals


def exchange(arrays, p, plans):
    """Send every face to its neighbour and receive theirs (gloo p2p)."""
    import torch
    import torch.distributed as dist
    reqs, recvs = [], []
    for d in range(4):
        q = p["nbr"][d]
        if q < 0:
            continue
        for t, A in enumerate(arrays):
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(face(A, p, d))), q,
                                   tag=d * 8 + t))
        # from the neighbour in direction d: it sent in direction d^1
        nq = plans[q]
        for t, A in enumerate(arrays):
            fl = nq["face_hi"][d ^ 1] - nq["face_lo"][d ^ 1] + 1
            buf = torch.empty((fl,) + A.shape[2:], dtype=torch.float64)
            recvs.append((dist.irecv(buf, q, tag=(d ^ 1) * 8 + t), A, nq, d ^ 1, buf))
    for r in reqs:
        r.wait()
    for r, A, nq, d, buf in recvs:
        r.wait()
        put(A, nq, d, nq["send_slot"][d], buf.numpy())


def _worker(rank, world, port, shape, grid, steps, consts, result_q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nx, ny, nz = shape
        px, py = grid
        cfg = W.GridConfig(nx=nx, ny=ny, nz=nz, **consts)
        g = O.grid_from(cfg)
        plans = [W.plan(cfg, px, py, r) for r in range(world)]
        p = plans[rank]
        rng = np.random.default_rng(1802)
        n3, n2 = O.shapes(g)
        s0 = O.State(rng.uniform(150, 350, n3), rng.uniform(150, 350, n3),
                     rng.uniform(150, 350, n2), rng.uniform(150, 350, n2))
        G = s0.energy.reshape((nx + 2, ny + 2, nz), order="F")
        GS = s0.energy_surf.reshape((nx + 2, ny + 2), order="F")
        GB = s0.energy_pbl.reshape((nx + 2, ny + 2), order="F")
        o = 1
        lnx, lny = p["lnx"], p["lny"]
        E = np.full((lnx + 4, lny + 4, nz), np.nan)
        SF = np.full((lnx + 4, lny + 4), np.nan)
        PB = np.full((lnx + 4, lny + 4), np.nan)
        i0 = 0 if p["own_w"] else 1
        i1 = lnx + 1 if p["own_e"] else lnx
        j0 = 0 if p["own_s"] else 1
        j1 = lny + 1 if p["own_n"] else lny
        gi, gj = slice(p["gi0"] + i0, p["gi0"] + i1 + 1), slice(p["gj0"] + j0, p["gj0"] + j1 + 1)
        li, lj = slice(i0 + o, i1 + 1 + o), slice(j0 + o, j1 + 1 + o)
        E[li, lj] = G[gi, gj]
        SF[li, lj] = GS[gi, gj]
        PB[li, lj] = GB[gi, gj]
        exchange([E, SF[:, :, None], PB[:, :, None]], p, plans)
        EU = None
        for _ in range(steps):
            U, P = local_step(E, SF, PB, p, g)
            EU = P
            exchange([U], p, plans)
            E = U
        pieces = (gi, gj, E[li, lj].copy(), EU[li, lj].copy())
        out = [None] * world if rank == 0 else None
        dist.gather_object(pieces, out, dst=0)
        if rank == 0:
            want = O.COracle().steps(g, s0, steps)
            We = want.energy.reshape((nx + 2, ny + 2, nz), order="F")
            Wu = want.energy_u.reshape((nx + 2, ny + 2, nz), order="F")
            got_e = np.full_like(We, np.nan)
            got_u = np.full_like(Wu, np.nan)
            for (a, b, e, u) in out:
                got_e[a, b] = e
                got_u[a, b] = u
            result_q.put((bool(np.array_equal(got_e, We)), bool(np.array_equal(got_u, Wu)),
                          int(np.sum(got_e != We))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("shape,grid,steps", [
    ((17, 13, 5), (2, 1), 3), ((17, 13, 5), (1, 2), 3), ((16, 16, 8), (2, 2), 4),
    ((17, 13, 5), (3, 2), 3), ((33, 29, 11), (2, 4), 2)])
def test_decomposed_run_matches_oracle_bitwise(shape, grid, steps):
    import torch.multiprocessing as mp
    world = grid[0] * grid[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    consts = dict(diffusion_velocity=0.125, radiation_intensity=0.37, transfer_velocity=0.013)
    procs = [ctx.Process(target=_worker,
                         args=(r, world, port, shape, grid, steps, consts, q))
             for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=240)
    assert all(pr.exitcode == 0 for pr in procs), [pr.exitcode for pr in procs]
    same_e, same_u, nbad = q.get(timeout=5)
    assert same_e and same_u, f"{nbad} cells differ"



# ---------------------------------------------------------------------------
# the decomposed TWO-STEP pass (weather_pair.cuh, dist mode), restated in numpy:
# 2-deep faces, 1-deep far slots to wrap partners, one corner column to each
# diagonal neighbour (hftw_plan depth / diag / diag_slot), the halo
# intermediates computed with the inner rule, ghost finals from the wrap
# partners' published intermediates.  NaN halos poison any read of a slot the
# plan does not fill.
# ---------------------------------------------------------------------------
def plan_writes(A, p, kind):
    """Every halo write my owned cells produce under the two-step plan:
    (target rank, kind, target local i, target local j, values over k)."""
    o, nx, ny = 1, p["lnx"], p["lny"]
    i0 = 0 if p["own_w"] else 1
    i1 = nx + 1 if p["own_e"] else nx
    j0 = 0 if p["own_s"] else 1
    j1 = ny + 1 if p["own_n"] else ny
    out = []
    for d in range(4):
        q = p["nbr"][d]
        if q < 0:
            continue
        for layer in range(1, p["depth"][d] + 1):
            slot = p["send_slot"][d] + (layer - 1) * (1 if d in (W_, S_) else -1)
            if d in (W_, E_):
                li = layer if d == W_ else nx + 1 - layer
                for lj in range(j0, j1 + 1):
                    out.append((q, kind, slot, lj, A[li + o, lj + o].copy()))
            else:
                lj = layer if d == S_ else ny + 1 - layer
                for li in range(i0, i1 + 1):
                    out.append((q, kind, li, slot, A[li + o, lj + o].copy()))
    for c in range(4):
        q = p["diag"][c]
        if q < 0:
            continue
        li, lj = (nx if c & 1 else 1), (ny if c & 2 else 1)
        out.append((q, kind, p["diag_slot"][c][0], p["diag_slot"][c][1], A[li + o, lj + o].copy()))
    return out


def apply_writes(arrays, rank, all_writes):
    for writes in all_writes:
        for (q, kind, ti, tj, v) in writes:
            if q == rank:
                arrays[kind][ti + 1, tj + 1] = v


def stencil(P, nx, ny, g):
    """Inner rule (weather.cpp:130-150) at every local (i, j) in [0, nx+1] x [0, ny+1]."""
    dv = g.diffusion_velocity
    c5, c6 = 1 - 5.0 * dv, 1 - 6.0 * dv
    C = P[1:nx + 3, 1:ny + 3]
    s = P[0:nx + 2, 1:ny + 3] + P[2:nx + 4, 1:ny + 3]
    s = s + P[1:nx + 3, 0:ny + 2]
    s = s + P[1:nx + 3, 2:ny + 4]
    U = np.empty_like(C)
    U[:, :, 1:-1] = c6 * C[:, :, 1:-1] + dv * ((s[:, :, 1:-1] + C[:, :, :-2]) + C[:, :, 2:])
    U[:, :, 0] = c5 * C[:, :, 0] + dv * (s[:, :, 0] + C[:, :, 1])
    U[:, :, -1] = c5 * C[:, :, -1] + dv * (s[:, :, -1] + C[:, :, -2])
    out = np.full_like(P, np.nan)
    out[1:nx + 3, 1:ny + 3] = U
    return out


def ghost_rules(U, P, p, g, far_cols=None, far_rows=None):
    """Overwrite the OWNED ghost cells of U with the cyclic rules
    (weather.cpp:152-168, i ghosts last) from P; the partner values come from
    P's far slots or, for finals, from the wrap partners' published columns."""
    o, nx, ny = 1, p["lnx"], p["lny"]
    c2, dv = 1 - 2.0 * g.diffusion_velocity, g.diffusion_velocity
    J = slice(1 + o, ny + 1 + o)
    if p["own_s"]:
        far = P[:, p["sfar"] + o] if far_rows is None else far_rows["s"]
        U[1 + o:nx + 1 + o, o] = (c2 * P[1 + o:nx + 1 + o, o] +
                                  dv * (far[1 + o:nx + 1 + o] + P[1 + o:nx + 1 + o, 1 + o]))
    if p["own_n"]:
        far = P[:, p["nfar"] + o] if far_rows is None else far_rows["n"]
        U[1 + o:nx + 1 + o, ny + 1 + o] = (c2 * P[1 + o:nx + 1 + o, ny + 1 + o] +
                                           dv * (P[1 + o:nx + 1 + o, ny + o] +
                                                 far[1 + o:nx + 1 + o]))
    j0 = 0 if p["own_s"] else 1
    j1 = ny + 1 if p["own_n"] else ny
    Jo = slice(j0 + o, j1 + 1 + o)
    if p["own_w"]:
        far = P[p["wfar"] + o] if far_cols is None else far_cols["w"]
        U[o, Jo] = c2 * P[o, Jo] + dv * (P[1 + o, Jo] + far[Jo])
    if p["own_e"]:
        far = P[p["efar"] + o] if far_cols is None else far_cols["e"]
        U[nx + 1 + o, Jo] = c2 * P[nx + 1 + o, Jo] + dv * (far[Jo] + P[nx + o, Jo])
    del J
    return U


def _pair_worker(rank, world, port, shape, grid, passes, consts, result_q, pform=False):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nx_g, ny_g, nz = shape
        px, py = grid
        cfg = W.GridConfig(nx=nx_g, ny=ny_g, nz=nz, **consts)
        g = O.grid_from(cfg)
        plans = [W.plan(cfg, px, py, r) for r in range(world)]
        p = plans[rank]
        rng = np.random.default_rng(1802)
        n3, n2 = O.shapes(g)
        s0 = O.State(rng.uniform(150, 350, n3), rng.uniform(150, 350, n3),
                     rng.uniform(150, 350, n2), rng.uniform(150, 350, n2))
        G = s0.energy.reshape((nx_g + 2, ny_g + 2, nz), order="F")
        GS = s0.energy_surf.reshape((nx_g + 2, ny_g + 2), order="F")
        GB = s0.energy_pbl.reshape((nx_g + 2, ny_g + 2), order="F")
        o, nx, ny = 1, p["lnx"], p["lny"]
        E = np.full((nx + 4, ny + 4, nz), np.nan)
        SF = np.full((nx + 4, ny + 4, 1), np.nan)
        PB = np.full((nx + 4, ny + 4, 1), np.nan)
        i0 = 0 if p["own_w"] else 1
        i1 = nx + 1 if p["own_e"] else nx
        j0 = 0 if p["own_s"] else 1
        j1 = ny + 1 if p["own_n"] else ny
        gi, gj = slice(p["gi0"] + i0, p["gi0"] + i1 + 1), slice(p["gj0"] + j0, p["gj0"] + j1 + 1)
        li, lj = slice(i0 + o, i1 + 1 + o), slice(j0 + o, j1 + 1 + o)
        E[li, lj] = G[gi, gj]
        SF[li, lj, 0] = GS[gi, gj]
        PB[li, lj, 0] = GB[gi, gj]

        def exchange_all(named):
            mine = []
            for kind, A in named.items():
                mine += plan_writes(A, p, kind)
            allw = [None] * world
            dist.all_gather_object(allw, mine)
            apply_writes(named, rank, allw)

        exchange_all({"e": E, "sf": SF, "pb": PB})
        for t in range(passes):
            # pform: the passes after the first read a post-physics field and all but
            # the last store one (the library's PIN / POUT); the halos carry it too
            P = E if pform and t > 0 else phys(E, SF[:, :, 0], PB[:, :, 0], g)
            U1 = ghost_rules(stencil(P, nx, ny, g), P, p, g)    # intermediate on [0, n+1]^2
            P1 = phys(U1, SF[:, :, 0], PB[:, :, 0], g)          # P' (post-physics)
            U2 = np.full_like(E, np.nan)
            U2[1 + o:nx + 1 + o, 1 + o:ny + 1 + o] = stencil(P1, nx, ny, g)[
                1 + o:nx + 1 + o, 1 + o:ny + 1 + o]             # inner finals
            # ghost finals: the wrap partners publish P' at their columns 1 / nx
            # (rows 1 / ny) -- gathered here, read by the partner
            pub = {"c1": P1[1 + o].copy(), "cn": P1[nx + o].copy(),
                   "r1": P1[:, 1 + o].copy(), "rn": P1[:, ny + o].copy()}
            allpub = [None] * world
            dist.all_gather_object(allpub, pub)
            wrap = lambda d: p["nbr"][d] if (p["nbr"][d] >= 0 and p["depth"][d] == 1) else rank
            far_cols = {"w": allpub[wrap(W_)]["cn"], "e": allpub[wrap(E_)]["c1"]}
            far_rows = {"s": allpub[wrap(S_)]["rn"], "n": allpub[wrap(N_)]["r1"]}
            U2 = ghost_rules(U2, P1, p, g, far_cols, far_rows)
            if pform and t + 1 < passes:
                U2 = phys(U2, SF[:, :, 0], PB[:, :, 0], g)
            own = np.full_like(E, np.nan)
            own[li, lj] = U2[li, lj]
            E = own
            exchange_all({"e": E})
        pieces = (gi, gj, E[li, lj].copy())
        out = [None] * world if rank == 0 else None
        dist.gather_object(pieces, out, dst=0)
        if rank == 0:
            want = O.COracle().steps(g, s0, 2 * passes)
            We = want.energy.reshape((nx_g + 2, ny_g + 2, nz), order="F")
            got = np.full_like(We, np.nan)
            for (a, b, e) in out:
                got[a, b] = e
            result_q.put((bool(np.array_equal(got, We)), int(np.sum(~(got == We)))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("shape,grid,passes,pform", [
    ((17, 13, 5), (2, 1), 2, False), ((17, 13, 5), (1, 2), 2, False),
    ((16, 16, 8), (2, 2), 2, False), ((17, 13, 5), (3, 2), 2, False),
    ((33, 29, 11), (2, 4), 1, False), ((21, 19, 4), (3, 3), 2, False),
    # the field kept post-physics between the passes of one call
    ((17, 13, 5), (2, 1), 3, True), ((16, 16, 8), (2, 2), 3, True),
    ((21, 19, 4), (3, 3), 2, True)])
def test_decomposed_pair_pass_matches_oracle_bitwise(shape, grid, passes, pform):
    import torch.multiprocessing as mp
    world = grid[0] * grid[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    consts = dict(diffusion_velocity=0.125, radiation_intensity=0.37, transfer_velocity=0.013)
    procs = [ctx.Process(target=_pair_worker,
                         args=(r, world, port, shape, grid, passes, consts, q, pform))
             for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=240)
    assert all(pr.exitcode == 0 for pr in procs), [pr.exitcode for pr in procs]
    same, nbad = q.get(timeout=5)
    assert same, f"{nbad} cells differ"
