"""K1 (rf_analytic, FP32) us per 128-channel row block at N = 2048 / 4096 / 8192."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2507_15464_b200 as tb

for n, rows in ((2048, 64 * 64), (4096, 64 * 128), (8192, 16 * 192)):
    x = torch.randn((rows, n), device="cuda")
    out = torch.empty((rows, n), dtype=torch.complex64, device="cuda")
    for _ in range(3):
        tb.rf_analytic(x, "f32", out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        tb.rf_analytic(x, "f32", out=out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"N={n}: {ms * 1e3 / rows:.4f} us/row  {rows * n * 12 / ms / 1e6:.0f} GB/s (f32 in + c64 out)", flush=True)
