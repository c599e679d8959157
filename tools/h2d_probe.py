"""Probe host->device copy bandwidth on the GPU box (pinned, 1D vs 2D pitched)."""
import torch, time
n, m = 262144, 5000
h = torch.empty(n * m, dtype=torch.int8).pin_memory()
d = torch.empty(n * 5008, dtype=torch.int8, device="cuda")
s = torch.cuda.Stream()
import ctypes
cudart = ctypes.CDLL("libcudart.so.12") if False else None
def t(fn, reps=5):
    torch.cuda.synchronize(); fn(); torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
ms = t(lambda: d[: n * m].copy_(h, non_blocking=True))
print("1D pinned H2D %.1f GB/s" % (n * m / ms / 1e6))
hv = h.view(n, m); dv = d.view(n, 5008)[:, :m]
ms = t(lambda: dv.copy_(hv, non_blocking=True))
print("2D pinned H2D (torch) %.1f GB/s" % (n * m / ms / 1e6))
# two streams, halves
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def two():
    half = n * m // 2
    with torch.cuda.stream(s1): d[:half].copy_(h[:half], non_blocking=True)
    with torch.cuda.stream(s2): d[half:n*m].copy_(h[half:], non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
ms = t(two)
print("1D pinned H2D 2 streams %.1f GB/s" % (n * m / ms / 1e6))
