#!/usr/bin/env python3
"""Measure the B200 machine-table entries the paper's model needs
(perfmodel.hpp:19-33) on the GPU box and write profiles/machine_b200.json.

  bw_htod : pinned host->device cudaMemcpy, 1 GiB            (GB/s)
  ra_d    : device random 8-byte read-modify-write updates   (GUP/s)
  bw_h1c  : host copy bandwidth, one core (numpy)            (GB/s, read+write)
  ra_h    : host random 8-byte updates, one core (numpy)     (GUP/s)
Machine characterisation only -- not part of the hot path.
"""
import json
import os
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def cuda_time(fn, reps=5):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        s.record()
        fn()
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e) * 1e-3)
    return best


def main():
    dev = torch.device("cuda:0")
    n = 1 << 27  # 1 GiB of fp64
    h = torch.empty(n, dtype=torch.float64, pin_memory=True)
    d = torch.empty(n, dtype=torch.float64, device=dev)
    t = cuda_time(lambda: d.copy_(h, non_blocking=True))
    bw_htod = n * 8 / t / 1e9
    # device random access: index_add_ of random 8-byte updates into a 4 GiB table
    table = torch.zeros(1 << 29, dtype=torch.float64, device=dev)
    m = 1 << 26
    idx = torch.randint(0, table.numel(), (m,), device=dev)
    vals = torch.ones(m, dtype=torch.float64, device=dev)
    t = cuda_time(lambda: table.index_add_(0, idx, vals))
    ra_d = m / t / 1e9
    # host, one core
    a = np.ones(1 << 26)
    b = np.empty_like(a)
    t0 = time.perf_counter()
    for _ in range(3):
        np.copyto(b, a)
    bw_h1c = 3 * 2 * a.nbytes / (time.perf_counter() - t0) / 1e9
    tab = np.zeros(1 << 26)
    hi = np.random.default_rng(0).integers(0, tab.size, 1 << 24)
    t0 = time.perf_counter()
    np.add.at(tab, hi, 1.0)
    ra_h = hi.size / (time.perf_counter() - t0) / 1e9
    out = {"bw_htod": bw_htod, "ra_d": ra_d, "bw_h1c": bw_h1c, "ra_h": ra_h,
           "source": "tools/measure_machine.py on the GPU box (pinned 1 GiB H2D; index_add_ "
                     "2^26 random fp64 updates into 4 GiB; numpy 1-core copy and add.at)",
           "host_nproc": os.cpu_count(), "gpu": torch.cuda.get_device_name(0)}
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "machine_b200.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
