import torch
B, nz, nx = 256, 2048, 1024
g = torch.randn((B, nz, nx), device="cuda"); y = torch.empty_like(g)
for _ in range(3): y.copy_(g)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): y.copy_(g)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"torch copy {ms:.3f} ms -> {2 * g.numel() * 4 / ms / 1e6:.0f} GB/s")
