"""PCIe probe 2: the e2e pipeline's D2H shapes (2D row-block copies) vs 1D copies,
one vs two D2H streams, with and without a concurrent H2D stream.

The ASUCA host field is (nx+2)(ny+2)nz fp64 with i fastest; a row block of `nj` rows is
nz runs of nj*(nx+2)*8 contiguous bytes, (nx+2)(ny+2)*8 apart.
"""
import time
import torch
from cuda.bindings import runtime as rt

nx, ny, nz = 1581, 1301, 58
NB = 32
rowb = (nx + 2) * 8
plane = rowb * (ny + 2)
n = plane * nz // 8
H = [torch.empty(n, dtype=torch.float64, pin_memory=True) for _ in range(3)]
D = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(3)]
S = [torch.cuda.Stream() for _ in range(3)]
D2H = rt.cudaMemcpyKind.cudaMemcpyDeviceToHost
H2D = rt.cudaMemcpyKind.cudaMemcpyHostToDevice
rows = [((ny + 2) * b // NB, (ny + 2) * (b + 1) // NB) for b in range(NB)]


def t(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best


def blk2d(h, d, r0, r1, kind, s):
    # device staging dense per block (like hftw_step_host): block b lives at d + r0*rowb*nz
    w = (r1 - r0) * rowb
    hp = h.data_ptr() + r0 * rowb
    dp = d.data_ptr() + r0 * rowb * nz
    if kind == D2H:
        err, = rt.cudaMemcpy2DAsync(hp, plane, dp, w, w, nz, kind, s.cuda_stream)
    else:
        err, = rt.cudaMemcpy2DAsync(dp, w, hp, plane, w, nz, kind, s.cuda_stream)
    assert err == rt.cudaError_t.cudaSuccess, err


def blk1d(h, d, r0, r1, kind, s):
    off = r0 * rowb * nz
    nb = (r1 - r0) * rowb * nz
    if kind == D2H:
        err, = rt.cudaMemcpyAsync(h.data_ptr() + off, d.data_ptr() + off, nb, kind, s.cuda_stream)
    else:
        err, = rt.cudaMemcpyAsync(d.data_ptr() + off, h.data_ptr() + off, nb, kind, s.cuda_stream)
    assert err == rt.cudaError_t.cudaSuccess, err


gb = n * 8 / 1e9


def run(copy, arrays, streams_of, h2d=False):
    def f():
        if h2d:
            for (r0, r1) in rows:
                copy(H[2], D[2], r0, r1, H2D, S[2])
        for b, (r0, r1) in enumerate(rows):
            for a in arrays:
                copy(H[a], D[a], r0, r1, D2H, S[streams_of(a, b)])
    return f


res = {}
for name, copy in (("1d", blk1d), ("2d", blk2d)):
    res[name + " d2h 1 field"] = gb / t(run(copy, [0], lambda a, b: 0))
    res[name + " d2h 2 fields 1 stream"] = 2 * gb / t(run(copy, [0, 1], lambda a, b: 0))
    res[name + " d2h 2 fields 2 streams (per field)"] = 2 * gb / t(run(copy, [0, 1], lambda a, b: a))
    res[name + " d2h 2 fields 2 streams (alt blocks)"] = 2 * gb / t(run(copy, [0, 1], lambda a, b: b & 1))
    res[name + " d2h 2 fields + h2d 1 field: d2h-equivalent"] = 2 * gb / t(
        run(copy, [0, 1], lambda a, b: a, h2d=True))
    res[name + " h2d 1 field"] = gb / t(lambda: [copy(H[2], D[2], r0, r1, H2D, S[2]) for (r0, r1) in rows])
for k, v in res.items():
    print(f"{k:50s} {v:6.1f} GB/s")
