"""Small driver for ncu: one cfg2 DAS chunk (K1 + K2) and one row-operator launch.

  python tools/profile_kernels.py [--iters 2]
  ncu --set full -k regex:"das_image|analytic|rowconv" -c 3 python tools/profile_kernels.py --frames 64 --maps 256
"""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2507_15464_b200 as tb  # noqa: E402
from bench import CFG2, frame_scatterers, grid  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=1)
ap.add_argument("--frames", type=int, default=8)
ap.add_argument("--maps", type=int, default=32)
ap.add_argument("--map-shape", default="2048x1024", help="depth x lateral of the row-operator maps (cfg2: 512x256)")
args = ap.parse_args()

cfg = CFG2
F = args.frames
sx, sz, a = frame_scatterers(cfg, range(F))
rf = tb.synthesize_batch(sx, sz, a, angles=[0.0], n_el=cfg["n_el"], pitch=cfg["pitch"], fs=cfg["fs"],
                         c=cfg["c"], f0=cfg["f0"], fbw=cfg["fbw"], n_samples=cfg["n_samples"])
x, z = grid(cfg)
plan = tb.plane_wave_plan(n_el=cfg["n_el"], pitch=cfg["pitch"], fs=cfg["fs"], c=cfg["c"],
                          n_samples=cfg["n_samples"], x=x, z=z, f_number=cfg["f_number"])
an = torch.empty((F, 1, cfg["n_el"], cfg["n_samples"]), dtype=torch.complex64, device="cuda")
img = torch.empty((F, cfg["nz"], cfg["nx"]), device="cuda")
gen = torch.Generator(device="cuda").manual_seed(1)
mz, mx = (int(v) for v in args.map_shape.split("x"))
maps = (torch.rand((args.maps, mz, mx), device="cuda", generator=gen) < 0.02).float()
K = torch.randn((mz, 129), device="cuda", generator=gen)
y = torch.empty_like(maps)
z4 = np.linspace(5e-3, 45e-3, 2048)
dx4 = 38.4e-3 / 1023
pk = dict(n_el=cfg["n_el"], pitch=cfg["pitch"], fs=cfg["fs"], c=cfg["c"], f0=cfg["f0"], fbw=cfg["fbw"],
          f_number=cfg["f_number"], n_samples=cfg["n_samples"])
torch.cuda.synchronize()
for _ in range(args.iters):
    tb.rf_analytic(rf, "f32", out=an, sample_range=plan.sample_range())  # as das_image calls it
    tb.das_from_analytic(an, plan, out=img)
    tb.tidas_rowconv(maps, K, out=y)
    tb.build_row_kernels(z4, 129, dx4, neighbourhood=8, **pk)  # K5 at cfg4
torch.cuda.synchronize()
print("ok", float(img.sum()), float(y.abs().sum()))
