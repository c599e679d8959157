"""Measured int8 tensor-core peak on this GPU via cuBLASLt (torch._int_mm),
the library reference the cross-term kernel's roofline is compared with."""
import torch
for n in (8192, 16384):
    a = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda")
    b = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda").t()
    for _ in range(3):
        torch._int_mm(a, b)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(10):
        e0.record(); torch._int_mm(a, b); e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"cublas int8 {n}^3: {2 * n**3 / best / 1e9:.0f} TOPS ({best:.3f} ms)")
    a16 = torch.randn(n, n, dtype=torch.bfloat16, device="cuda")
    torch.matmul(a16, a16)
    best = 1e9
    for _ in range(10):
        e0.record(); torch.matmul(a16, a16); e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"cublas bf16 {n}^3: {2 * n**3 / best / 1e9:.0f} TFLOPS")
