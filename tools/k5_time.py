import sys, time, torch, numpy as np
sys.path.insert(0, '.')
import paper_2507_15464_b200 as tb
from tests.setups import CFG4, CFG2
for cfg in (CFG2, CFG4):
    x, z = np.linspace(*cfg["x"], cfg["nx"]), np.linspace(*cfg["z"], cfg["nz"])
    kw = dict(n_el=cfg["n_el"], pitch=cfg["pitch"], fs=cfg["fs"], c=cfg["c"], f0=cfg["f0"], fbw=cfg["fbw"], f_number=cfg["f_number"], n_samples=cfg["n_samples"])
    for _ in range(2): tb.build_row_kernels(z, 129, x[1]-x[0], **kw)
    torch.cuda.synchronize(); e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): tb.build_row_kernels(z, 129, x[1]-x[0], **kw)
    e1.record(); torch.cuda.synchronize(); print(cfg["nz"], "rows K5 ms", e0.elapsed_time(e1)/5)
