"""Bitwise comparison of DAS images between kernel variants (cfg2 grid, a ragged
grid and a coarse grid whose windows overflow the staging boxes; 61 frames):
  python tools/das_dump.py /tmp/a.npz [lib.so]            # write
  python tools/das_dump.py /tmp/b.npz [lib.so] /tmp/a.npz # write and compare with a"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2507_15464_b200 import _lib  # noqa: E402

if len(sys.argv) > 2:
    _lib.load(Path(sys.argv[2]))
import bench  # noqa: E402
import paper_2507_15464_b200 as tb  # noqa: E402

res = {}
cfg = bench.CFG2
x, z = bench.grid(cfg)
sx, sz, a = bench.frame_scatterers(cfg, range(64))
kw = {k: cfg[k] for k in ("n_el", "pitch", "fs", "c", "f0", "fbw", "n_samples")}
rf = tb.synthesize_batch(sx, sz, a, angles=[0.0], dtype=torch.float32, **kw)
for name, (xx, zz) in {"cfg2": (x, z), "ragged": (x[:250], z[:500]), "coarse": (x[::4], z[::3])}.items():
    plan = tb.plane_wave_plan(n_el=cfg["n_el"], pitch=cfg["pitch"], fs=cfg["fs"], c=cfg["c"],
                              n_samples=cfg["n_samples"], x=xx, z=zz, f_number=cfg["f_number"])
    res[name] = tb.das_image(rf[:61], plan).cpu().numpy()  # 61: a partial frame batch at the end
    res[name + "_window"] = np.array(plan.window())
np.savez(sys.argv[1], **res)
if len(sys.argv) > 3:
    ref = np.load(sys.argv[3])
    for k, v in res.items():
        r = ref[k]
        diff = int((v != r).sum()) if v.shape == r.shape else -1
        rel = float(np.abs(v - r).max() / max(np.abs(r).max(), 1e-30)) if v.shape == r.shape else float("nan")
        print(f"{k}: shape {v.shape} differing elements {diff} max rel diff {rel:.3g}")
else:
    print("written", {k: v.shape for k, v in res.items()})
