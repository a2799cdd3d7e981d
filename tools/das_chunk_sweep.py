"""cfg2 DAS (K1 + K2) over 256 frames at different chunk sizes (frames per
K1 / K2 launch): small chunks keep the analytic intermediate L2-resident
(less DRAM traffic), large chunks shorten the kernels' last-wave tails.
python tools/das_chunk_sweep.py [--sustain] [--lib=variant.so] [chunk ...]
--sustain: 1.5 s of load before a 1 s timed window (the bench's power-capped
steady state) and the median SM clock over the window (NVML)."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2507_15464_b200 import _lib  # noqa: E402

_libs = [a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--lib=")]
if _libs:  # a variant library (tools/build_variant.sh)
    _lib.load(Path(_libs[0]))
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
sustain = "--sustain" in sys.argv
chunks = [int(c) for c in sys.argv[1:] if not c.startswith("--")] or [8, 16, 24, 32, 64, 128, 256]


def sm_clock_sampler():
    import threading
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    samples, stop = [], threading.Event()

    def run():
        while not stop.is_set():
            samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
            stop.wait(0.05)
    th = threading.Thread(target=run, daemon=True)
    th.start()
    return samples, stop, th
ref_img = None
for ch in chunks:
    plan = tb.plane_wave_plan(n_el=cfg["n_el"], pitch=cfg["pitch"], fs=cfg["fs"], c=cfg["c"],
                              n_samples=cfg["n_samples"], x=x, z=z, f_number=cfg["f_number"])
    plan.chunk_bytes = ch * 128 * 4096 * 8
    ws = imaging.DasWorkspace(plan)
    assert ws.chunk == ch, ws.chunk
    for _ in range(3):
        tb.das_image(rf, plan, out=img, workspace=ws)
    torch.cuda.synchronize()
    if ref_img is None:
        ref_img = img.clone()
    same = bool(torch.equal(img, ref_img))  # images are bitwise independent of the chunk size
    n_it, clk = 10, None
    if sustain:
        import statistics
        import time
        t0 = time.perf_counter()
        while time.perf_counter() - t0 < 1.5:
            tb.das_image(rf, plan, out=img, workspace=ws)
            torch.cuda.synchronize()
        n_it = 600
        samples, stop, th = sm_clock_sampler()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n_it):
        tb.das_image(rf, plan, out=img, workspace=ws)
    e1.record()
    torch.cuda.synchronize()
    if sustain:
        stop.set()
        th.join()
        clk = statistics.median(samples) if samples else None
    us = e0.elapsed_time(e1) / n_it / F * 1e3
    print(json.dumps({"chunk_frames": ch, "us_per_frame": us, "frames_per_s": 1e6 / us, "sm_mhz": clk,
                      "bitwise_equal_to_first": same}), flush=True)
    del ws
