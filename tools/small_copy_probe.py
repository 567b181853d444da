"""Floor for a 68 MB sweep (34 MB read + 34 MB write): torch copy, 6 buffer pairs round robin."""
import torch
n = 256 * 256 * 64 + 2 * 256 * 64  # ~34 MB of fp64
pairs = [(torch.rand(n, dtype=torch.float64, device="cuda"), torch.empty(n, dtype=torch.float64, device="cuda")) for _ in range(6)]
for i in range(12):
    s, d = pairs[i % 6]; d.copy_(s)
torch.cuda.synchronize()
evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(120)]
for i, (a, b) in enumerate(evs):
    s, d = pairs[i % 6]
    a.record(); d.copy_(s); b.record()
torch.cuda.synchronize()
t = sorted(a.elapsed_time(b) for a, b in evs)
print(f"torch copy 2 x {n*8/1e6:.1f} MB: median {t[len(t)//2]*1e3:.1f} us, min {t[0]*1e3:.1f} us -> {2*n*8/(t[len(t)//2]*1e-3)/1e9:.0f} GB/s")
