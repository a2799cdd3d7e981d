"""Throughput of the DAS path at the other BASELINE.json configs (1 GPU).

  python tools/bench_configs.py [--steps 10] [--warmup 3] [--configs cfg1,cfg3,cfg5]

Each line: frames/s of K1 + K2 with the RF resident in HBM (CUDA events around
`das_image`), per-frame algorithmic bytes (RF in its arrival dtype
+ FP32 image) and the HBM-roofline fraction. Inputs are seeded synthetic frames
simulated on the device (cfg5: scaled to std 1000, rounded, clipped to int16).
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2507_15464_b200 as tb  # noqa: E402
from paper_2507_15464_b200 import imaging  # noqa: E402

HBM = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] if (ROOT / "MEASURED_PEAKS.json").exists() else 6650.0

CFGS = {
    "cfg1": dict(n_el=64, pitch=0.3e-3, f0=5e6, fs=20e6, fbw=0.6, N=2048, nz=256, nx=128, z=(5e-3, 40e-3),
                 x=(-9.6e-3, 9.6e-3), angles=[0.0], frames=256, n_scat=1, dtype=torch.float64, out="envelope",
                 bytes=64 * 2048 * 8 + 256 * 128 * 4, region=None),
    "cfg3": dict(n_el=128, pitch=0.3e-3, f0=5e6, fs=40e6, fbw=0.6, N=4096, nz=1024, nx=512, z=(5e-3, 45e-3),
                 x=(-19.2e-3, 19.2e-3), angles=list(np.deg2rad(np.linspace(-10, 10, 11))), frames=64,
                 n_scat=2000, n_bright=5, dtype=torch.float32, out="coherent",
                 bytes=11 * 128 * 4096 * 4 + 1024 * 512 * 4, region=((-20e-3, 20e-3), (5e-3, 45e-3))),
    "cfg5": dict(n_el=192, pitch=0.3e-3, f0=5e6, fs=40e6, fbw=0.6, N=8192, nz=1024, nx=1024, z=(5e-3, 60e-3),
                 x=(-28.8e-3, 28.8e-3), angles=[0.0], frames=64, n_scat=4000, dtype=torch.int16, out="envelope",
                 bytes=192 * 8192 * 2 + 1024 * 1024 * 4, region=((-28.8e-3, 28.8e-3), (5e-3, 60e-3))),
}


def make_rf(name, c):
    F = c["frames"]
    rng = np.random.default_rng(7)
    if name == "cfg1":  # single point scatterer (0, 20 mm), replicated frames
        sx, sz, a = np.zeros((F, 1)), np.full((F, 1), 20e-3), np.ones((F, 1))
    else:
        (x0, x1), (z0, z1) = c["region"]
        S = c["n_scat"] + c.get("n_bright", 0)
        sx = rng.uniform(x0, x1, (F, S))
        sz = rng.uniform(z0, z1, (F, S))
        a = rng.standard_normal((F, S))
        if c.get("n_bright"):
            a[:, c["n_scat"]:] = 20.0  # bright point targets
    # cfg5: simulated in float32, each frame scaled to std 1000, rounded, clipped (library quantiser)
    return tb.synthesize_batch(sx, sz, a, angles=c["angles"], n_el=c["n_el"], pitch=c["pitch"], fs=c["fs"],
                               c=1540.0, f0=c["f0"], fbw=c["fbw"], n_samples=c["N"], dtype=c["dtype"],
                               target_std=1000.0)


def run_configs(names, steps=10, warmup=3, echo=False):
    """Frames/s of das_image (K1 + K2, RF resident) per config; returns {name: record}."""
    res = {}
    for name in names:
        c = CFGS[name]
        rf = make_rf(name, c)
        x, z = np.linspace(*c["x"], c["nx"]), np.linspace(*c["z"], c["nz"])
        plan = tb.plane_wave_plan(n_el=c["n_el"], pitch=c["pitch"], fs=c["fs"], c=1540.0, n_samples=c["N"],
                                  x=x, z=z, angles=c["angles"], f_number=1.5, out=c["out"])
        ws = imaging.DasWorkspace(plan)
        img = torch.empty((rf.shape[0], c["nz"], c["nx"]), device="cuda")
        for _ in range(warmup):
            tb.das_image(rf, plan, out=img, workspace=ws)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            tb.das_image(rf, plan, out=img, workspace=ws)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        fps = rf.shape[0] / (ms / 1e3)
        gbs = c["bytes"] * fps / 1e9
        res[name] = {"frames_per_step": int(rf.shape[0]), "ms_per_step": ms, "frames_per_s": fps,
                     "bytes_per_frame": c["bytes"], "hbm_GBps": gbs, "hbm_frac": gbs / HBM,
                     "rf_dtype": str(c["dtype"]).replace("torch.", ""), "transmits": len(c["angles"]),
                     "grid": [c["nz"], c["nx"]], "out": c["out"], "chunk_frames": ws.chunk,
                     "checksum": float(img.double().sum())}
        if echo:
            print(json.dumps({name: res[name]}), flush=True)
        del rf, img, ws
        torch.cuda.empty_cache()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--configs", default="cfg1,cfg3,cfg5")
    args = ap.parse_args()
    print(json.dumps(run_configs(args.configs.split(","), args.steps, args.warmup, echo=True)))


if __name__ == "__main__":
    main()
