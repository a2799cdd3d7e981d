"""Check + time the tensor-core row operator against the oracle and the CUDA-core path."""
import os, subprocess, sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2507_15464_b200 as tb
from oracle import tidas as ot, das as od

rng = np.random.default_rng(0)
for (B, nz, nx, T) in [(128, 3, 256, 129), (40, 5, 100, 129), (64, 4, 64, 31), (200, 3, 1024, 1), (256, 2, 1024, 129)]:
    g = ((rng.random((B, nz, nx)) < 0.2) * rng.standard_normal((B, nz, nx))).astype(np.float32)
    K = rng.standard_normal((nz, T)).astype(np.float32)
    gd, Kd = torch.as_tensor(g).cuda(), torch.as_tensor(K).cuda()
    y = tb.tidas_rowconv(gd, Kd)
    a = tb.tidas_rowconv_adjoint(gd, Kd)
    torch.cuda.synchronize()
    e1 = od.rel_l2(y.cpu().numpy(), ot.rowconv_fwd(g, K))
    e2 = od.rel_l2(a.cpu().numpy(), ot.rowconv_adj(g, K))
    print(f"B={B} nz={nz} nx={nx} T={T}: fwd rel_l2 {e1:.2e} adj rel_l2 {e2:.2e}", flush=True)

# timing at cfg4 size
B, nz, nx, T = 256, 2048, 1024, 129
gen = torch.Generator(device="cuda").manual_seed(1)
g = (torch.rand((B, nz, nx), device="cuda", generator=gen) < 0.02).float() * torch.randn((B, nz, nx), device="cuda", generator=gen)
K = torch.randn((nz, T), device="cuda", generator=gen) / 16
y = torch.empty_like(g)
for _ in range(2): tb.tidas_rowconv(g, K, out=y)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5): tb.tidas_rowconv(g, K, out=y)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(f"cfg4 fwd {ms:.3f} ms  -> {B * nz * nx * 8 / ms / 1e6:.0f} GB/s", flush=True)
# compare with the CUDA-core path on a slice
ys = torch.empty_like(g[:8])
env = dict(os.environ)
print("checksum tc", float(y[:8].double().abs().sum()))
