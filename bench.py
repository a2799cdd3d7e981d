#!/usr/bin/env python
"""Benchmark of the DAS / tiDAS hot path (BASELINE.json metric).

  python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1], the headline): cfg2 — 128-channel x 4096
float32 RF frames of seeded speckle (2000 scatterers, 0-degree plane wave) ->
512 x 256 DAS images (Hann F#1.5, linear interpolation, envelope). A step is
one pass of the hot path over F frames per GPU (default 64, 128 MiB of RF —
larger than L2, so no flush is needed between steps). ``value`` is frames/s of
the whole job with inputs resident in HBM; ``e2e`` runs the public API
(``HostPipeline.run``) from pinned host RF to pinned host images with every
H2D / D2H copy inside the timed region (copies overlap the kernels on three
streams; the line reports the measured H2D ceiling it is bound by).
Under torchrun (N > 1) frames are sharded (weak scaling) and the images are
all-gathered over NCCL inside the step. The JSON line also reports the tiDAS
row operator (cfg2 maps, and cfg4 forward + adjoint) in ``tidas``.

``--impl reference`` times the reference's own CPU algorithm (oracle port,
oracle/cpu_bench.py) on this host's cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "DAS/tiDAS frames/s (128 ch, 512x256 px) and % of HBM-bandwidth roofline"
BYTES_PER_FRAME_CFG2 = 128 * 4096 * 4 + 512 * 256 * 4          # 2,621,440
BYTES_PER_MAP_CFG2 = 512 * 256 * 4 * 2                         # 1,048,576
BYTES_PER_MAP_CFG4 = 2048 * 1024 * 4 * 2                       # 16,777,216

CFG2 = dict(n_el=128, pitch=0.3e-3, f0=5e6, fs=40e6, c=1540.0, fbw=0.6, n_samples=4096,
            nz=512, nx=256, z=(5e-3, 45e-3), x=(-19.2e-3, 19.2e-3), f_number=1.5, n_scat=2000,
            region_x=(-20e-3, 20e-3), region_z=(5e-3, 45e-3))
CFG4 = dict(nz=2048, nx=1024, taps=129, maps=256, density=0.02)


def committed_traffic():
    """DRAM bytes per frame of K1 + K2 from the committed ncu --set full capture
    (profiles/*/traffic.json, written by tools/traffic_from_ncu.py), or None."""
    for p in sorted(ROOT.glob("profiles/*/traffic.json"), reverse=True):
        try:
            return json.loads(p.read_text())
        except (OSError, ValueError):
            continue
    return None


WORKLOAD = ("cfg2 (BASELINE.json configs[1]): DAS, 128 ch x 4096 f32 RF -> 512x256 px, Hann F#1.5, "
            "linear interp, envelope")


def k2_live_pairs(cfg, x, z) -> int:
    """(pixel, channel) pairs inside the Hann F# aperture of pixels whose t*
    lies on the trace — the gathers K2 must do per frame and transmit."""
    xs = (np.arange(-cfg["n_el"] // 2, cfg["n_el"] // 2) + 0.5) * cfg["pitch"]
    Z, X = np.meshgrid(np.asarray(z, float), np.asarray(x, float), indexing="ij")
    live = (np.abs(xs[None, None, :] - X[..., None]) < (Z / (2.0 * cfg["f_number"]))[..., None]).sum(-1)
    pos = 2.0 * Z / cfg["c"] * cfg["fs"]  # 0-degree plane wave: t* = 2 z / c
    return int((live * ((pos >= 0) & (pos <= cfg["n_samples"] - 1))).sum())


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if self.proc is None or not self.path:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = []
        for line in Path(self.path).read_text().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6 and parts[0].isdigit():
                rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [int(r[0]) for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": int(rows[0][1]),
                "reasons": reasons, "samples": len(rows)}


def grid(cfg):
    return np.linspace(*cfg["x"], cfg["nx"]), np.linspace(*cfg["z"], cfg["nz"])


def frame_scatterers(cfg, frames, seed=2025):
    """Seeded per-frame speckle: frame f uses default_rng(seed + f) (global index)."""
    sx = np.empty((len(frames), cfg["n_scat"]))
    sz = np.empty_like(sx)
    a = np.empty_like(sx)
    for k, f in enumerate(frames):
        rng = np.random.default_rng(seed + int(f))
        sx[k] = rng.uniform(*cfg["region_x"], cfg["n_scat"])
        sz[k] = rng.uniform(*cfg["region_z"], cfg["n_scat"])
        a[k] = rng.standard_normal(cfg["n_scat"])
    return sx, sz, a


def cpu_baseline(budget_pixels: int, workers=None, target_s: float = 0.0):
    """Reference algorithm (oracle port) on a bounded pixel sample of one cfg2 frame.

    With ``target_s`` > 0 a first small sample sizes a second one to about
    ``target_s`` seconds of CPU work, which is the one reported."""
    from oracle import cpu_bench, geom, simulate as osim
    cfg = CFG2
    sx, sz, a = frame_scatterers(cfg, [0])
    rf = osim.synthesize(sx[0], sz[0], a[0], n_el=cfg["n_el"], pitch=cfg["pitch"], fs=cfg["fs"],
                         c=cfg["c"], f0=cfg["f0"], fbw=cfg["fbw"], n_samples=cfg["n_samples"],
                         tx=("plane", 0.0)).astype(np.float32).astype(np.float64)
    x, z = grid(cfg)
    ts = geom.plane_wave_expected_arrival(x[None, :], z[:, None], 0.0, cfg["n_el"], cfg["pitch"], cfg["c"])
    kw = dict(fs=cfg["fs"], c=cfg["c"], pitch=cfg["pitch"], f_number=cfg["f_number"], x=x, z=z,
              t_star=ts, workers=workers)
    pps, n, dt, w = cpu_bench.pixels_per_second(rf, n_pixels=budget_pixels, **kw)
    if target_s > 0:
        n2 = int(min(max(budget_pixels, pps * target_s), cfg["nx"] * cfg["nz"]))
        pps, n, dt, w = cpu_bench.pixels_per_second(rf, n_pixels=n2, seed=1, **kw)
    return pps / (cfg["nx"] * cfg["nz"]), n, dt, w


def run_reference(args):
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return 0
    workers = os.cpu_count() or 1
    px_per_step = max(workers * 96, 256)
    vals = []
    for k in range(args.warmup + args.steps):
        fps, n, dt, w = cpu_baseline(px_per_step, workers)
        if k >= args.warmup:
            vals.append((fps, dt))
    fps = statistics.median(v[0] for v in vals)
    ms = 1e3 * statistics.median(v[1] for v in vals)
    sample = f"{px_per_step} seeded pixels of one cfg2 frame per step, extrapolated to 131072 px/frame"
    line = {"impl": "reference", "metric": METRIC, "value": fps, "unit": "frames/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: seeded speckle, 2000 scatterers, 0-degree plane wave (oracle simulator)",
            "config": {"workload": WORKLOAD, "device": "cpu (host cores, oracle port of the reference algorithm)"},
            "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": workers, "kind": "port",
                             "sample": sample},
            "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--frames", type=int, default=64, help="cfg2 frames per GPU per step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-tidas", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the cfg1 / cfg3 / cfg5 DAS lines")
    ap.add_argument("--cpu-pixels", type=int, default=0, help="cpu_baseline pixel sample (0 = auto)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    import paper_2507_15464_b200 as tb
    from paper_2507_15464_b200 import imaging, parallel

    rank, world = parallel.init()
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if args.warmup < 3:
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)

    cfg = CFG2
    F = args.frames
    total_frames = F * world
    fa, fb = parallel.shard_range(total_frames, rank, world)
    frames = list(range(fa, fb))
    x, z = grid(cfg)
    sx, sz, amp = frame_scatterers(cfg, frames)
    rf = tb.synthesize_batch(sx, sz, amp, angles=[0.0], n_el=cfg["n_el"], pitch=cfg["pitch"],
                             fs=cfg["fs"], c=cfg["c"], f0=cfg["f0"], fbw=cfg["fbw"],
                             n_samples=cfg["n_samples"], dtype=torch.float32, device=dev)
    plan = tb.plane_wave_plan(n_el=cfg["n_el"], pitch=cfg["pitch"], fs=cfg["fs"], c=cfg["c"],
                              n_samples=cfg["n_samples"], x=x, z=z, angles=[0.0],
                              f_number=cfg["f_number"], device=dev)
    ws = imaging.DasWorkspace(plan, dev)
    img = torch.empty((len(frames), cfg["nz"], cfg["nx"]), device=dev)
    gathered = torch.empty((total_frames, cfg["nz"], cfg["nx"]), device=dev) if world > 1 else None
    stream = torch.cuda.current_stream()

    def step():
        if world == 1:
            tb.das_image(rf, plan, out=img, workspace=ws)
        else:
            # 16-frame sub-chunks: the all-gather of chunk c (async NCCL over
            # NVLink) overlaps the K1 + K2 of chunk c + 1
            parallel.pipelined_gather(
                lambda c0, c1: tb.das_image(rf[c0:c1], plan, out=img[c0:c1], workspace=ws),
                len(frames), gathered, sub=16)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v):
        if world > 1:
            t = torch.tensor([v], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return float(t.item())
        return v

    for _ in range(args.warmup):
        step()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        barrier()
    clocks = clk.summary()
    ms_total = max_over_ranks(e0.elapsed_time(e1))
    ms_step = ms_total / args.steps
    value = total_frames / (ms_step / 1e3)
    if world == 1:
        launches = args.steps * imaging.launches_per_call(len(frames), plan, ws)
    else:
        launches = args.steps * sum(imaging.launches_per_call(min(16, len(frames) - c0), plan, ws)
                                    for c0 in range(0, len(frames), 16))

    # ---- per-kernel timing of one step (roofline of the DAS pipeline K1 + K2)
    chunk = ws.chunk
    k1_ms, k2_ms = [], []
    for _ in range(3):
        for f0 in range(0, len(frames), chunk):
            f1 = min(len(frames), f0 + chunk)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            an = ws.buf[: f1 - f0]
            ev[0].record(stream)
            tb.rf_analytic(rf[f0:f1], plan.prec, out=an)
            ev[1].record(stream)
            tb.das_from_analytic(an, plan, out=img[f0:f1])
            ev[2].record(stream)
            torch.cuda.synchronize()
            k1_ms.append(ev[0].elapsed_time(ev[1]) / (f1 - f0))
            k2_ms.append(ev[1].elapsed_time(ev[2]) / (f1 - f0))
    k1 = statistics.median(k1_ms)
    k2 = statistics.median(k2_ms)
    hbm, peak_kind = peaks()
    pipe_gbs = BYTES_PER_FRAME_CFG2 / ((k1 + k2) / 1e3) / 1e9
    tr = committed_traffic()
    traffic = tr["das_pipeline_bytes_per_frame"] * chunk if tr else None
    roofline = {"bound": "hbm", "achieved": pipe_gbs, "peak": hbm, "unit": "GB/s",
                "frac": pipe_gbs / hbm, "traffic": traffic,
                "traffic_source": tr.get("source") if tr else None,
                "kernel": f"das pipeline per chunk of {chunk} frames: tidas_rf_analytic (K1) + "
                          "das_image_kernel (K2)",
                "bytes_per_launch": BYTES_PER_FRAME_CFG2 * chunk, "peak_source": peak_kind,
                "per_frame_us": {"K1_analytic": k1 * 1e3, "K2_das": k2 * 1e3}}
    # K2's binding resource is shared memory: every live (pixel, channel) pair
    # gathers 3 complex64 samples (24 B) per frame from the staged window
    pairs = k2_live_pairs(cfg, x, z)
    smem_peak = 148 * 128 * (clocks.get("sm_mhz") or 1965) * 1e6 / 1e9  # GB/s, 128 B/clk/SM
    smem_ach = pairs * 24 / (k2 * 1e-3) / 1e9
    k2_smem = {"bound": "smem", "achieved": smem_ach, "peak": smem_peak, "unit": "GB/s",
               "frac": smem_ach / smem_peak, "live_pairs_per_frame": pairs,
               "bytes_per_pair": 24, "kernel": "das_image_kernel (K2)",
               "note": "shared-memory gather roofline of K2 (128 B/clk/SM at the measured SM clock); "
                       "the HBM roofline above is the contract metric"}

    # ---- e2e through the public API with pinned host buffers: HostPipeline
    # (H2D of chunk i+1 || K1 + K2 of chunk i || D2H of chunk i-1, three streams)
    host_rf = torch.empty(rf.shape, dtype=torch.float32, pin_memory=True)
    host_rf.copy_(rf)
    host_img = torch.empty(img.shape, dtype=torch.float32, pin_memory=True)
    pipe = tb.HostPipeline(plan, chunk=16)
    for _ in range(max(1, min(args.warmup, 3))):
        pipe.run(host_rf, host_img)
    pipe.synchronize()
    barrier()
    e0.record(stream)
    pipe.wait_for(stream)
    for _ in range(args.steps):
        pipe.run(host_rf, host_img)
    pipe.join(stream)
    e1.record(stream)
    barrier()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1)) / args.steps
    # the PCIe ceiling: a bare pinned H2D copy of one step's RF
    rf_dev = torch.empty_like(rf)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(5):
        rf_dev.copy_(host_rf, non_blocking=True)
    t1.record(stream)
    torch.cuda.synchronize()
    h2d_gbs = host_rf.numel() * 4 * 5 / t0.elapsed_time(t1) / 1e6
    e2e = {"value": total_frames / (e2e_ms / 1e3), "unit": "frames/s",
           "h2d_bytes_per_step": int(host_rf.numel() * 4), "d2h_bytes_per_step": int(host_img.numel() * 4),
           "ms_per_step": e2e_ms, "api": "HostPipeline.run (pinned host RF -> pinned host images), chunk 16",
           "bound": {"kind": "pcie_h2d", "h2d_GBps_measured": h2d_gbs,
                     "frac": host_rf.numel() * 4 / (e2e_ms / 1e3) / 1e9 / h2d_gbs}}
    launches_e2e = args.steps * pipe.launches(len(frames))
    del rf_dev

    # ---- tiDAS row operator: cfg2 maps (forward) and cfg4 (forward + adjoint)
    tidas = None
    if not args.no_tidas:
        dx = x[1] - x[0]
        K2d, _ = tb.build_row_kernels(z, 129, dx, n_el=cfg["n_el"], pitch=cfg["pitch"], fs=cfg["fs"],
                                      c=cfg["c"], f0=cfg["f0"], fbw=cfg["fbw"], f_number=cfg["f_number"],
                                      n_samples=cfg["n_samples"], neighbourhood=8)
        gen = torch.Generator(device=dev).manual_seed(7 + rank)
        # 512 cfg2 maps per step: 256 MiB in + 256 MiB out, larger than L2 (no flush needed)
        M2 = 512
        maps2 = (torch.rand((M2, cfg["nz"], cfg["nx"]), device=dev, generator=gen) < 0.02).float() * \
            torch.randn((M2, cfg["nz"], cfg["nx"]), device=dev, generator=gen)
        out2 = torch.empty_like(maps2)
        for _ in range(args.warmup):
            tb.tidas_rowconv(maps2, K2d, out=out2)
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            tb.tidas_rowconv(maps2, K2d, out=out2)
        e1.record(stream)
        barrier()
        t2 = max_over_ranks(e0.elapsed_time(e1)) / args.steps
        g2 = (BYTES_PER_MAP_CFG2 * M2 + K2d.numel() * 4) / (t2 / 1e3) / 1e9
        del maps2, out2
        # cfg4: 256 maps of 2048 x 1024, forward + adjoint per step
        c4 = CFG4
        M = c4["maps"]
        K4 = torch.randn((c4["nz"], c4["taps"]), device=dev, generator=gen) / 16
        maps4 = (torch.rand((M, c4["nz"], c4["nx"]), device=dev, generator=gen) < c4["density"]).float() * \
            torch.randn((M, c4["nz"], c4["nx"]), device=dev, generator=gen)
        y4 = torch.empty_like(maps4)
        a4 = torch.empty_like(maps4)
        for _ in range(max(1, min(args.warmup, 3))):
            tb.tidas_rowconv(maps4, K4, out=y4)
            tb.tidas_rowconv_adjoint(y4, K4, out=a4)
        barrier()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        fw, ad = [], []
        for _ in range(max(3, min(args.steps, 10))):
            ev[0].record(stream)
            tb.tidas_rowconv(maps4, K4, out=y4)
            ev[1].record(stream)
            tb.tidas_rowconv_adjoint(y4, K4, out=a4)
            ev[2].record(stream)
            torch.cuda.synchronize()
            fw.append(ev[0].elapsed_time(ev[1]))
            ad.append(ev[1].elapsed_time(ev[2]))
        tf, ta = max_over_ranks(statistics.median(fw)), max_over_ranks(statistics.median(ad))
        g4 = (BYTES_PER_MAP_CFG4 * M + K4.numel() * 4) / (tf / 1e3) / 1e9
        cpu_rowconv = None
        if rank == 0 and world == 1 and not args.no_cpu_baseline:
            # the row operator's float64 CPU restatement (no reference counterpart,
            # SURVEY §8(d)), one process, on a bounded sample of one cfg4 map
            sys.path.insert(0, str(ROOT))
            from oracle import tidas as ot
            rows = 128
            g1 = maps4[0, :rows].double().cpu().numpy()[None]
            K1h = K4[:rows].double().cpu().numpy()
            t0 = time.perf_counter()
            ot.rowconv_fwd(g1, K1h)
            ct = time.perf_counter() - t0
            cpu_rowconv = {"kind": "port (restatement)", "cores": 1, "unit": "maps/s (fwd)",
                           "value": rows / c4["nz"] / ct, "sample": f"{rows} of {c4['nz']} rows of one cfg4 map"}
        tidas = {
            "cfg2_fwd": {"value": M2 * world / (t2 / 1e3), "unit": "maps/s", "maps_per_step_per_gpu": M2,
                         "ms_per_step": t2,
                         "roofline": {"bound": "hbm", "achieved": g2, "peak": hbm, "unit": "GB/s",
                                      "frac": g2 / hbm, "traffic": None,
                                      "kernel": "rowconv_tc1_kernel<fwd> (tcgen05 3xTF32)"}},
            "cfg4_fwd_adj": {"value": M * world / ((tf + ta) / 1e3), "unit": "maps/s (fwd+adj)",
                             "fwd_ms": tf, "adj_ms": ta, "maps_per_gpu": M,
                             "roofline": {"bound": "hbm", "achieved": g4, "peak": hbm, "unit": "GB/s",
                                          "frac": g4 / hbm,
                                          "traffic": (tr or {}).get("rowconv_cfg4_bytes_per_launch"),
                                          "kernel": "rowconv_tc1_kernel<fwd> (tcgen05 3xTF32), 256 maps/launch"}},
            "cpu_baseline": cpu_rowconv,
            "row_kernels": "K5 build_row_kernels, cfg2 geometry, 129 taps, neighbourhood 8 (cfg2); "
                           "seeded random K for cfg4 timing",
        }
        del maps4, y4, a4

    # ---- the paper's "600 points in 600 configurations" error
    # sweep (theta + local / global error matrices), default probe
    sweep = None
    if rank == 0 and not args.no_tidas:
        eps = float(np.load(ROOT / "tests/golden/ref_vectors.npz")["eps"])
        d600 = np.linspace(0.005, 0.042, 600)
        run = lambda: tb.error_sweep(d600, tb.ProbeConfig(), tb.Kossoff(0.6), tb.FNumber(1.0),  # noqa: E731
                                     tx_focus_depth=25e-3, window_half_width=eps)
        run()
        torch.cuda.synchronize()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        th600, _, _ = run()
        s1.record(stream)
        torch.cuda.synchronize()
        sec = s0.elapsed_time(s1) / 1e3
        sweep = {"cells": 360000, "seconds": sec, "cells_per_s": 360000 / sec,
                 "finite_cells": int(np.isfinite(th600).sum()),
                 "paper_cpu_minutes": {"das": 28.35, "tidas": 21.11},
                 "api": "error_sweep (theta, local and global error matrices of run_error_sweep), "
                        "600 scatterer depths x 600 reference profiles, 5-42 mm, 7 MHz, Tx focus 25 mm",
                 "timing": "CUDA events around the public call (host geometry + D2H of the matrices inside)"}
        if world == 1 and not args.no_cpu_baseline:
            # the same sweep's CPU algorithm (oracle port of tidas.py / experiments.py,
            # pinned to the reference's CSV fixtures), one process, on a bounded
            # 12 x 12 sample of the grid, extrapolated per cell
            sys.path.insert(0, str(ROOT))
            from oracle import theta as oth
            probe = dict(n_el=192, pitch=0.2e-3, f0=7e6, fs=50e6, c=1540.0, fbw=0.75)
            d12 = d600[::50]
            t0 = time.perf_counter()
            oth.error_sweep(d12, d12, probe, tx_focus=25e-3, half_width=eps)
            ct = time.perf_counter() - t0
            sweep["cpu_baseline"] = {"kind": "port", "cores": 1, "sample": f"{len(d12)} x {len(d12)} cells",
                                     "seconds_per_cell": ct / len(d12) ** 2,
                                     "extrapolated_600x600_minutes": ct / len(d12) ** 2 * 360000 / 60}

    # ---- the other BASELINE.json DAS configs (1 GPU, RF resident; parity-tested
    # in tests/test_gpu_das.py): cfg1 f64 PSF, cfg3 11-angle coherent, cfg5 int16
    others = None
    if rank == 0 and world == 1 and not args.no_configs:
        sys.path.insert(0, str(ROOT / "tools"))
        import bench_configs
        others = {k: {"frames_per_s": v["frames_per_s"], "ms_per_step": v["ms_per_step"],
                      "frames_per_step": v["frames_per_step"], "hbm_frac": v["hbm_frac"],
                      "bytes_per_frame": v["bytes_per_frame"], "rf_dtype": v["rf_dtype"],
                      "transmits": v["transmits"], "grid": v["grid"], "out": v["out"]}
                  for k, v in bench_configs.run_configs(["cfg1", "cfg3", "cfg5"]).items()}
        others["note"] = ("das_image (K1 + K2) with the RF resident in HBM, CUDA events over 10 steps; "
                          "cfg5 timed on 64 of its 1024 frames per step")

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        workers = os.cpu_count() or 1
        n_px = args.cpu_pixels or max(workers * 48, 96)
        fps, n, dt, w = cpu_baseline(n_px, workers, target_s=0.0 if args.cpu_pixels else 8.0)
        cpu = {"value": fps, "unit": "frames/s", "cores": w, "kind": "port",
               "sample": f"{n} seeded pixels of one cfg2 frame ({dt:.1f} s over {w} processes), "
                         "reference per-pixel algorithm (full-trace shifts + Hilbert), "
                         "extrapolated to 131072 px/frame"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic: seeded speckle (2000 N(0,1) scatterers over 40x40 mm per frame), "
                    "0-degree plane-wave RF simulated on the device (float32)",
            "config": {"workload": WORKLOAD,
                       "frames_per_step_per_gpu": F, "parallelism": f"frame-sharded dp{world}",
                       "l2": "inputs larger than L2 (128 MiB RF per GPU per step)",
                       "gather": "NCCL all_gather of images inside the step, pipelined per 16 frames with the "
                                 "DAS of the next 16" if world > 1 else "none"},
            "roofline": roofline, "k2_smem_roofline": k2_smem, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches,
            "gpu_launches_e2e": launches_e2e,
            "clocks": clocks, "tidas": tidas, "theta_error_sweep": sweep, "other_configs": others,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
