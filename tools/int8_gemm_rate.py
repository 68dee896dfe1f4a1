"""Dense INT8 GEMM rate of this B200 through cuBLASLt (torch._int_mm, tcgen05 kind::i8 path) next
to FP64 (torch.matmul float64, DMMA): the ratio that bounds an Ozaki-style FP64 emulation of the
pair kernel's GEMMs. usage: python tools/int8_gemm_rate.py"""
import torch


def rate(fn, flops, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return flops * reps / (e0.elapsed_time(e1) / 1e3) / 1e12


for n in (4096, 8192, 16384):
    a = torch.randint(-127, 127, (n, n), dtype=torch.int8, device="cuda")
    b = torch.randint(-127, 127, (n, n), dtype=torch.int8, device="cuda").t().contiguous().t()
    r8 = rate(lambda: torch._int_mm(a, b), 2.0 * n ** 3)
    x = torch.randn(n, n, dtype=torch.float64, device="cuda")
    r64 = rate(lambda: x @ x, 2.0 * n ** 3, reps=3 if n > 8192 else 10)
    print(f"n={n}: int8 {r8:.0f} TOPS, fp64 {r64:.1f} TFLOP/s, ratio {r8 / r64:.0f}")
