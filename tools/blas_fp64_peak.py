"""cuBLAS DGEMM / ZGEMM throughput via torch (FP64 library reference for the roofline)."""
import torch

def bench(dtype, n, flop_per_mac):
    a = torch.randn(n, n, dtype=dtype, device="cuda")
    b = torch.randn(n, n, dtype=dtype, device="cuda")
    for _ in range(3):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    reps = 10
    e0.record()
    for _ in range(reps):
        torch.matmul(a, b)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"{dtype} n={n}: {ms:.3f} ms  {flop_per_mac * n**3 / ms / 1e9:.2f} TFLOP/s")

for n in (4096, 8192):
    bench(torch.float64, n, 2)
    bench(torch.complex128, n, 8)
