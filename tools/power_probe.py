"""Board power and SM clock (NVML) in the power-capped steady state of the cfg2
DAS kernels: K1 + K2, K1 alone, K2 alone (256 frames per call, 1.5 s of load
then a 1 s window).  python tools/power_probe.py [lib.so] [--rowconv]
(--rowconv: the cfg4 row operator instead, microseconds per map; --cfg5: the
cfg5 DAS path, 64 int16 frames per call)"""
import json
import statistics
import sys
import threading
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2507_15464_b200 as tb  # noqa: E402

import pynvml  # noqa: E402

LIB = [a for a in sys.argv[1:] if not a.startswith("--")]
if LIB:  # a variant library (tools/build_variant.sh)
    from paper_2507_15464_b200 import _lib
    _lib.load(Path(LIB[0]))

pynvml.nvmlInit()
H = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
cfg, F = bench.CFG2, 256
x, z = bench.grid(cfg)
sx, sz, a = bench.frame_scatterers(cfg, range(F))
rf = tb.synthesize_batch(sx, sz, a, angles=[0.0], dtype=torch.float32,
                         **{k: cfg[k] for k in ("n_el", "pitch", "fs", "c", "f0", "fbw", "n_samples")})
plan = tb.plane_wave_plan(n_el=cfg["n_el"], pitch=cfg["pitch"], fs=cfg["fs"], c=cfg["c"],
                          n_samples=cfg["n_samples"], x=x, z=z, f_number=cfg["f_number"])
an = tb.rf_analytic(rf, "f32")
img = torch.empty((F, cfg["nz"], cfg["nx"]), device="cuda")
limit_w = pynvml.nvmlDeviceGetEnforcedPowerLimit(H) / 1e3


def sample(stop, out):
    while not stop.is_set():
        out.append((pynvml.nvmlDeviceGetPowerUsage(H) / 1e3, pynvml.nvmlDeviceGetClockInfo(H, pynvml.NVML_CLOCK_SM)))
        stop.wait(0.05)


cases = [("K1+K2", lambda: tb.das_image(rf, plan, out=img)),
         ("K1", lambda: tb.rf_analytic(rf, "f32", out=an)),
         ("K2", lambda: tb.das_from_analytic(an, plan, out=img))]
if "--cfg5" in sys.argv:  # cfg5: 64 int16 frames of 192 x 8192 -> 1024 x 1024 (µs per frame)
    del rf, an, img
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    import numpy as np
    from bench_configs import CFGS, make_rf
    c5 = CFGS["cfg5"]
    F = 64
    rf = make_rf("cfg5", c5, list(range(F)))
    plan = tb.plane_wave_plan(n_el=c5["n_el"], pitch=c5["pitch"], fs=c5["fs"], c=1540.0, n_samples=c5["N"],
                              x=np.linspace(*c5["x"], c5["nx"]), z=np.linspace(*c5["z"], c5["nz"]),
                              f_number=1.5)
    an = tb.rf_analytic(rf, "f32")
    img = torch.empty((F, c5["nz"], c5["nx"]), device="cuda")
    cases = [("cfg5 K1+K2", lambda: tb.das_image(rf, plan, out=img)),
             ("cfg5 K1", lambda: tb.rf_analytic(rf, "f32", out=an)),
             ("cfg5 K2", lambda: tb.das_from_analytic(an, plan, out=img))]
if "--rowconv" in sys.argv:  # cfg4 row operator (256 maps): forward on sparse maps, adjoint on its dense output
    del rf, an, img
    g = torch.Generator(device="cuda").manual_seed(3)
    maps = (torch.rand((256, 2048, 1024), device="cuda", generator=g) < 0.02).float() * \
        torch.randn((256, 2048, 1024), device="cuda", generator=g)
    Kr = torch.randn((2048, 129), device="cuda", generator=g) / 16
    yv, av = torch.empty_like(maps), torch.empty_like(maps)
    tb.tidas_rowconv(maps, Kr, out=yv)
    F = 256  # per-call units: maps
    cases = [("rowconv fwd (cfg4, sparse maps)", lambda: tb.tidas_rowconv(maps, Kr, out=yv)),
             ("rowconv adj (cfg4, dense input)", lambda: tb.tidas_rowconv_adjoint(yv, Kr, out=av))]
for name, fn in cases:
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < 1.5:
        fn()
        torch.cuda.synchronize()
    s, stop = [], threading.Event()
    th = threading.Thread(target=sample, args=(stop, s), daemon=True)
    th.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 0
    e0.record()
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < 1.0:
        for _ in range(20):
            fn()
        n += 20
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    us = e0.elapsed_time(e1) / n / F * 1e3
    print(json.dumps({"kernels": name, "us_per_frame": round(us, 4), "power_w": round(statistics.median(p for p, _ in s), 1),
                      "sm_mhz": statistics.median(c for _, c in s), "power_limit_w": limit_w,
                      "joule_per_frame_mJ": round(statistics.median(p for p, _ in s) * us * 1e-3, 4)}), flush=True)
