"""PCIe probe: pinned H2D / D2H rates alone and concurrently (copy engines)."""
import time
import torch

n = 1 << 27  # 1 GiB of fp64
h1 = torch.empty(n, dtype=torch.float64, pin_memory=True)
h2 = torch.empty(n, dtype=torch.float64, pin_memory=True)
d1 = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best


gb = n * 8 / 1e9
h2d = t(lambda: d1.copy_(h1, non_blocking=True))
d2h = t(lambda: h2.copy_(d2, non_blocking=True))


def both():
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)


bt = t(both)


def d2h_two():
    with torch.cuda.stream(s1):
        h1[: n // 2].copy_(d1[: n // 2], non_blocking=True)
    with torch.cuda.stream(s2):
        h2[: n // 2].copy_(d2[: n // 2], non_blocking=True)


d2 = t(d2h_two)
print(f"H2D {gb/h2d:.1f} GB/s  D2H {gb/d2h:.1f} GB/s  concurrent H2D+D2H {2*gb/bt:.1f} GB/s total "
      f"({bt*1e3:.1f} ms for {gb:.2f}+{gb:.2f} GB)  two D2H streams {gb/d2:.1f} GB/s")
