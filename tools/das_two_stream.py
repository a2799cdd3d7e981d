"""cfg2 DAS with K1 of chunk c + 1 on a second stream beside K2 of chunk c
(ring of analytic buffers), in the power-capped steady state: 1.5 s of load,
then a 1 s timed window with the median SM clock (NVML).

  python tools/das_two_stream.py [chunk ...]      (default 16 32 64)

Small chunks keep the complex64 intermediate L2-resident (less DRAM traffic,
less power) and the concurrent kernels fill each other's last-wave tails."""
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

cfg, F = bench.CFG2, 256
x, z = bench.grid(cfg)
sx, sz, a = bench.frame_scatterers(cfg, range(F))
rf = tb.synthesize_batch(sx, sz, a, angles=[0.0], dtype=torch.float32,
                         **{k: cfg[k] for k in ("n_el", "pitch", "fs", "c", "f0", "fbw", "n_samples")})
plan = tb.plane_wave_plan(n_el=cfg["n_el"], pitch=cfg["pitch"], fs=cfg["fs"], c=cfg["c"],
                          n_samples=cfg["n_samples"], x=x, z=z, f_number=cfg["f_number"])
img = torch.empty((F, cfg["nz"], cfg["nx"]), device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream(priority=-1)


def clocks():
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


for ch in [int(c) for c in sys.argv[1:]] or [16, 32, 64]:
    nbuf = 3
    bufs = [torch.empty((ch, 1, cfg["n_el"], cfg["n_samples"]), dtype=torch.complex64, device="cuda")
            for _ in range(nbuf)]
    done_k1 = [torch.cuda.Event() for _ in range(nbuf)]
    done_k2 = [torch.cuda.Event() for _ in range(nbuf)]
    cur = torch.cuda.current_stream()

    def step():
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        n = F // ch
        for c in range(n):
            b = c % nbuf
            with torch.cuda.stream(s2):  # K1 of chunk c (after K2 of chunk c - nbuf released the buffer)
                if c >= nbuf:
                    s2.wait_event(done_k2[b])
                tb.rf_analytic(rf[c * ch:(c + 1) * ch], "f32", out=bufs[b])
                done_k1[b].record(s2)
            with torch.cuda.stream(s1):  # K2 of chunk c
                s1.wait_event(done_k1[b])
                tb.das_from_analytic(bufs[b], plan, out=img[c * ch:(c + 1) * ch])
                done_k2[b].record(s1)
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    t0 = time.perf_counter()
    while time.perf_counter() - t0 < 1.5:
        step()
        torch.cuda.synchronize()
    samples, stop, th = clocks()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n_it = 600
    e0.record()
    for _ in range(n_it):
        step()
    e1.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    us = e0.elapsed_time(e1) / n_it / F * 1e3
    print(json.dumps({"chunk_frames": ch, "two_streams": True, "us_per_frame": us, "frames_per_s": 1e6 / us,
                      "sm_mhz": statistics.median(samples) if samples else None,
                      "checksum": float(img.double().sum())}), flush=True)
    del bufs
