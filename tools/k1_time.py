"""Time K1 (rf_analytic) on 64 cfg2 frames."""
import sys, torch
sys.path.insert(0, ".")
import paper_2507_15464_b200 as tb
from bench import CFG2, frame_scatterers
cfg = CFG2; F = 64
sx, sz, a = frame_scatterers(cfg, range(F))
rf = tb.synthesize_batch(sx, sz, a, angles=[0.0], n_el=cfg["n_el"], pitch=cfg["pitch"], fs=cfg["fs"], c=cfg["c"], f0=cfg["f0"], fbw=cfg["fbw"], n_samples=cfg["n_samples"])
an = torch.empty(rf.shape, dtype=torch.complex64, device="cuda")
for _ in range(3): tb.rf_analytic(rf, "f32", out=an)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): tb.rf_analytic(rf, "f32", out=an)
e1.record(); torch.cuda.synchronize()
print("K1 us/frame", e0.elapsed_time(e1) * 1e3 / 10 / F, "checksum", float(an.abs().double().sum()))
