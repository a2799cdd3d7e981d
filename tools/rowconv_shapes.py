"""Row-operator bandwidth vs map count at fixed bytes (diagnoses page spread)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2507_15464_b200 as tb

for B, nz, nx in [(256, 2048, 1024), (128, 4096, 1024), (64, 8192, 1024), (32, 16384, 1024)]:
    gen = torch.Generator(device="cuda").manual_seed(1)
    g = torch.randn((B, nz, nx), device="cuda", generator=gen)
    K = torch.randn((nz, 129), device="cuda", generator=gen) / 16
    y = torch.empty_like(g)
    for _ in range(2): tb.tidas_rowconv(g, K, out=y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): tb.tidas_rowconv(g, K, out=y)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"B={B:4d} nz={nz:6d} nx={nx}: {ms:.3f} ms  {B * nz * nx * 8 / ms / 1e6:.0f} GB/s", flush=True)
    del g, y
