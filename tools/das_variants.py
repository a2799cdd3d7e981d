"""Time the DAS kernel (cfg2, 64 frames) for each TIDAS_DAS_VARIANT in a fresh process."""
import os, subprocess, sys
code = r'''
import sys, torch, numpy as np
sys.path.insert(0, ".")
import paper_2507_15464_b200 as tb
from paper_2507_15464_b200 import imaging
from bench import CFG2, frame_scatterers, grid
cfg = CFG2; F = 64
sx, sz, a = frame_scatterers(cfg, range(F))
rf = tb.synthesize_batch(sx, sz, a, angles=[0.0], n_el=cfg["n_el"], pitch=cfg["pitch"], fs=cfg["fs"], c=cfg["c"], f0=cfg["f0"], fbw=cfg["fbw"], n_samples=cfg["n_samples"])
x, z = grid(cfg)
plan = tb.plane_wave_plan(n_el=cfg["n_el"], pitch=cfg["pitch"], fs=cfg["fs"], c=cfg["c"], n_samples=cfg["n_samples"], x=x, z=z, f_number=cfg["f_number"])
an = tb.rf_analytic(rf, "f32")
img = torch.empty((F, cfg["nz"], cfg["nx"]), device="cuda")
for _ in range(3): tb.das_from_analytic(an, plan, out=img)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): tb.das_from_analytic(an, plan, out=img)
e1.record(); torch.cuda.synchronize()
print("us/frame", e0.elapsed_time(e1) * 1e3 / 10 / F, "checksum", float(img.double().sum()))
'''
for v in sys.argv[1:] or ["0", "55", "57", "58", "34"]:
    env = dict(os.environ, TIDAS_DAS_VARIANT=v)
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print("variant", v, (out.stdout.strip() or out.stderr.strip()[-400:]))
