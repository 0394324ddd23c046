"""Calibrate the roofline denominators MEASURED_PEAKS.json does not carry
(fp64 DGEMM, TF32, fp32 SIMT) plus host facts for the CPU baseline.
Run on the GPU box: python tools/calibrate_peaks.py > gpurun_out/peaks.json"""
import json, os, platform, subprocess, time
import torch

def bench_mm(dtype, n, tf32=False, iters=10):
    torch.backends.cuda.matmul.allow_tf32 = tf32
    a = torch.randn(n, n, device="cuda", dtype=dtype)
    b = torch.randn(n, n, device="cuda", dtype=dtype)
    for _ in range(3):
        a @ b
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(iters):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); a @ b; e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    return 2 * n**3 / best / 1e12

def bench_copy(nbytes=1 << 31):
    a = torch.empty(nbytes // 4, device="cuda", dtype=torch.float32).uniform_()
    b = torch.empty_like(a)
    for _ in range(3): b.copy_(a)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); b.copy_(a); e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    return 2 * nbytes / best / 1e9

def bench_h2d(nbytes=1 << 30):
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    d.copy_(h, non_blocking=True); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5): d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    return 5 * nbytes / (time.perf_counter() - t) / 1e9

out = {
    "fp64_tflops_cublas_8192": bench_mm(torch.float64, 8192, iters=5),
    "tf32_tflops_cublas_8192": bench_mm(torch.float32, 8192, tf32=True),
    "fp32_simt_tflops_cublas_8192": bench_mm(torch.float32, 8192, tf32=False),
    "bf16_tflops_cublas_8192": bench_mm(torch.bfloat16, 8192),
    "copy_gbs": bench_copy(),
    "h2d_pinned_gbs": bench_h2d(),
    "nproc": os.cpu_count(),
    "cpu": platform.processor(),
    "gpu": torch.cuda.get_device_name(0),
}
try:
    out["lscpu"] = subprocess.run(["lscpu"], capture_output=True, text=True).stdout[:1500]
    out["meminfo"] = open("/proc/meminfo").read()[:200]
except Exception as ex:
    out["err"] = str(ex)
print(json.dumps(out, indent=1))
