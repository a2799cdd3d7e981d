"""Row operator at small sizes: tcgen05 vs CUDA-core path."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2507_15464_b200 as tb

for B, nz, nx in ((64, 512, 256), (32, 512, 256), (256, 512, 256), (64, 2048, 1024), (32, 256, 128)):
    g = torch.randn((B, nz, nx), device="cuda")
    K = torch.randn((nz, 129), device="cuda")
    y = torch.empty_like(g)
    res = []
    for path in ("tensor", "simt"):
        for _ in range(3):
            tb.tidas_rowconv(g, K, out=y, path=path)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            tb.tidas_rowconv(g, K, out=y, path=path)
        e1.record()
        torch.cuda.synchronize()
        res.append(e0.elapsed_time(e1) / 20)
    gb = B * nz * nx * 8 / 1e9
    print(f"B={B} nz={nz} nx={nx}: tc {res[0]*1e3:.1f} us ({gb/res[0]*1e3:.0f} GB/s)  simt {res[1]*1e3:.1f} us "
          f"({gb/res[1]*1e3:.0f} GB/s)", flush=True)
