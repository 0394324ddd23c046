"""Measure cuBLAS DGEMM throughput (the fp64 DMMA roofline denominator)."""
import torch

for n in (4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        a @ b
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(5):
        e0.record(); a @ b; e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"dgemm {n}^3: {2 * n**3 / best / 1e9:.1f} TF/s ({best:.2f} ms)")
