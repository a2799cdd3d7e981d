"""cfg2 DAS (K1 + K2) over 256 frames at different chunk sizes (frames per
K1 / K2 launch): small chunks keep the analytic intermediate L2-resident
(less DRAM traffic), large chunks shorten the kernels' last-wave tails.
python tools/das_chunk_sweep.py [chunk ...]"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2507_15464_b200 as tb  # noqa: E402
from paper_2507_15464_b200 import imaging  # noqa: E402

cfg = bench.CFG2
F = 256
x, z = bench.grid(cfg)
sx, sz, a = bench.frame_scatterers(cfg, range(F))
rf = tb.synthesize_batch(sx, sz, a, angles=[0.0], dtype=torch.float32,
                         **{k: cfg[k] for k in ("n_el", "pitch", "fs", "c", "f0", "fbw", "n_samples")})
img = torch.empty((F, cfg["nz"], cfg["nx"]), device="cuda")
chunks = [int(c) for c in sys.argv[1:]] or [8, 16, 24, 32, 64, 128, 256]
for ch in chunks:
    plan = tb.plane_wave_plan(n_el=cfg["n_el"], pitch=cfg["pitch"], fs=cfg["fs"], c=cfg["c"],
                              n_samples=cfg["n_samples"], x=x, z=z, f_number=cfg["f_number"])
    plan.chunk_bytes = ch * 128 * 4096 * 8
    ws = imaging.DasWorkspace(plan)
    assert ws.chunk == ch, ws.chunk
    for _ in range(3):
        tb.das_image(rf, plan, out=img, workspace=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        tb.das_image(rf, plan, out=img, workspace=ws)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 10 / F * 1e3
    print(json.dumps({"chunk_frames": ch, "us_per_frame": us, "frames_per_s": 1e6 / us}), flush=True)
    del ws
