"""cfg2 K1 + K2 timing (256 frames, RF resident), optionally with a variant
library (tools/build_variant.sh): python tools/das_time.py [lib.so]"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2507_15464_b200 import _lib  # noqa: E402

if len(sys.argv) > 1:
    _lib.load(Path(sys.argv[1]))
import bench  # noqa: E402
import paper_2507_15464_b200 as tb  # noqa: E402

cfg, F = bench.CFG2, 256
x, z = bench.grid(cfg)
sx, sz, a = bench.frame_scatterers(cfg, range(F))
rf = tb.synthesize_batch(sx, sz, a, angles=[0.0], dtype=torch.float32,
                         **{k: cfg[k] for k in ("n_el", "pitch", "fs", "c", "f0", "fbw", "n_samples")})
plan = tb.plane_wave_plan(n_el=cfg["n_el"], pitch=cfg["pitch"], fs=cfg["fs"], c=cfg["c"], n_samples=cfg["n_samples"],
                          x=x, z=z, f_number=cfg["f_number"])
an = tb.rf_analytic(rf, "f32")
img = torch.empty((F, cfg["nz"], cfg["nx"]), device="cuda")


def t(fn, n=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n / F * 1e3


k2 = t(lambda: tb.das_from_analytic(an, plan, out=img))
both = t(lambda: tb.das_image(rf, plan, out=img))
print(json.dumps({"lib": sys.argv[1] if len(sys.argv) > 1 else "default", "K2_us": k2, "K1K2_us": both,
                  "fps": 1e6 / both, "checksum": float(img.double().sum())}), flush=True)
