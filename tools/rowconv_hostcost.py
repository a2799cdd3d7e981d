import sys, time, torch
sys.path.insert(0, ".")
import paper_2507_15464_b200 as tb
g = torch.randn((64, 512, 256), device="cuda"); K = torch.randn((512, 129), device="cuda"); y = torch.empty_like(g)
for _ in range(5): tb.tidas_rowconv(g, K, out=y)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(200): tb.tidas_rowconv(g, K, out=y)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host per call {1e6*(t1-t0)/200:.1f} us, wall per call {1e6*(t2-t0)/200:.1f} us")
