"""A/B timing of one library build (tools/build_variant.sh) on cfg2 and cfg1:
K1 over whole rows, K1 over the plan's sample range, K2 alone, K1 + K2 via
das_image (RF resident, 256 frames). Run once per library, alternating:
  python tools/ab_time.py [lib.so]"""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2507_15464_b200 import _lib  # noqa: E402

if len(sys.argv) > 1:
    _lib.load(Path(sys.argv[1]))
import bench  # noqa: E402
import paper_2507_15464_b200 as tb  # noqa: E402


def t(fn, F, n=20):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n / F * 1e3


res = {"lib": sys.argv[1] if len(sys.argv) > 1 else "default"}
cfg, F = bench.CFG2, 256
x, z = bench.grid(cfg)
sx, sz, a = bench.frame_scatterers(cfg, range(F))
rf = tb.synthesize_batch(sx, sz, a, angles=[0.0], dtype=torch.float32,
                         **{k: cfg[k] for k in ("n_el", "pitch", "fs", "c", "f0", "fbw", "n_samples")})
plan = tb.plane_wave_plan(n_el=cfg["n_el"], pitch=cfg["pitch"], fs=cfg["fs"], c=cfg["c"], n_samples=cfg["n_samples"],
                          x=x, z=z, f_number=cfg["f_number"])
an = tb.rf_analytic(rf, "f32")
img = torch.empty((F, cfg["nz"], cfg["nx"]), device="cuda")
rng = plan.sample_range() if hasattr(plan, "sample_range") else None
res["K1_full_us"] = t(lambda: tb.rf_analytic(rf, "f32", out=an), F)
if rng:
    res["K1_range_us"] = t(lambda: tb.rf_analytic(rf, "f32", out=an, sample_range=rng), F)
    res["range"] = list(rng)
res["K2_us"] = t(lambda: tb.das_from_analytic(an, plan, out=img), F)
res["pipe_us"] = t(lambda: tb.das_image(rf, plan, out=img), F)
res["checksum"] = float(img.double().sum())
del rf, an, img
# cfg1 (f64 RF, 2048 samples, 256 x 128 px)
sys.path.insert(0, str(Path(__file__).resolve().parent))
import bench_configs  # noqa: E402
c1 = bench_configs.CFGS["cfg1"]
rf1 = bench_configs.make_rf("cfg1", c1, list(range(256)))
x1, z1 = np.linspace(*c1["x"], c1["nx"]), np.linspace(*c1["z"], c1["nz"])
p1 = tb.plane_wave_plan(n_el=c1["n_el"], pitch=c1["pitch"], fs=c1["fs"], c=1540.0, n_samples=c1["N"], x=x1, z=z1)
img1 = torch.empty((256, c1["nz"], c1["nx"]), device="cuda")
res["cfg1_pipe_us"] = t(lambda: tb.das_image(rf1, p1, out=img1), 256)
print(json.dumps(res), flush=True)
