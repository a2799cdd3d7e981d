#!/usr/bin/env python
"""Benchmark of the DAS / tiDAS hot path (BASELINE.json metric).

  python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]

Headline workload (BASELINE.json configs[1]): cfg2 — 128-channel x 4096 float32
RF frames of seeded speckle (2000 scatterers, 0-degree plane wave) -> 512 x 256
DAS images (Hann F#1.5, linear interpolation, envelope). A step is one pass of
K1 + K2 over F frames per GPU (default 256: 512 MiB of RF, larger than L2, so
no flush is needed between steps). ``value`` is frames/s of the whole job with
the RF resident in HBM; ``e2e`` runs the public API (``HostPipeline.run``)
from pinned host RF to pinned host images with every H2D / D2H inside the
timed region.

Multi-GPU (north star (e)): ``--gpus N`` without torchrun re-launches itself
as N ranks under torch.distributed.run (127.0.0.1 rendezvous); under torchrun
WORLD_SIZE must equal N. Frames and maps are independent units, so every line
is frame- (map-) sharded with no data-path collective, except cfg3, whose
compounded images are gathered over NCCL inside the step as BASELINE.json's
cfg3 asks. cfg2 is weak-scaled (F frames per rank). ``other_configs`` adds
cfg1 (weak), cfg3 (64 frames, 11-angle coherent compounding, sharded + NCCL
image gather) and cfg5 (1024 int16 frames, sharded); ``tidas`` the row
operator (cfg2 maps, weak; cfg4's 256 maps and cfg5's 1024 maps sharded, K
built by K5 for each config's array and grid). NCCL's
communicator log is kept (NCCL_DEBUG=INFO to a file) and summarised.

``--impl reference`` times the reference's own CPU algorithm (oracle port,
oracle/cpu_bench.py) on this host's cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
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
CFG4 = dict(nz=2048, nx=1024, z=(5e-3, 45e-3), x=(-19.2e-3, 19.2e-3), taps=129, maps=256, density=0.02,
            neighbourhood=8)
# cfg5's tiDAS: the row operator on 1024 maps of the cfg5 grid (1024 x 1024, z 5-60 mm, x +-28.8 mm), K by K5
# for the cfg5 array (192 el, 0.3 mm, 5 MHz, 40 MHz, 8192 samples); maps drawn as cfg4's
CFG5T = dict(nz=1024, nx=1024, z=(5e-3, 60e-3), x=(-28.8e-3, 28.8e-3), taps=129, maps=1024, density=0.02,
             neighbourhood=8, probe=dict(n_el=192, pitch=0.3e-3, fs=40e6, c=1540.0, f0=5e6, fbw=0.6,
                                         f_number=1.5, n_samples=8192))
BYTES_PER_MAP_CFG5 = 1024 * 1024 * 4 * 2                       # 8,388,608
WORKLOAD = ("cfg2 (BASELINE.json configs[1]): DAS, 128 ch x 4096 f32 RF -> 512x256 px, Hann F#1.5, "
            "linear interp, envelope")
DATA = ("synthetic: seeded speckle (2000 N(0,1) scatterers over 40x40 mm per frame), 0-degree plane-wave RF "
        "(single-scattering model of simulate.py:193-259), float32")


def workload_config(frames_per_gpu: int, world: int) -> dict:
    """The workload identity both arms report (the reference arm's CPU sample
    is described in its cpu_baseline)."""
    return {"workload": WORKLOAD, "frames_per_step_per_gpu": frames_per_gpu,
            "parallelism": f"frame-sharded dp{world}",
            "l2": f"inputs larger than L2 ({frames_per_gpu * 2} MiB RF per GPU per step)",
            "gather": "none: cfg2 frames are independent units, each rank keeps the images it made (no data-path "
                      "collective); the NCCL image gather north star (e) asks for runs on cfg3's compounded "
                      "images (other_configs)" if world > 1 else "none"}


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def committed_traffic():
    """DRAM bytes of K1 + K2 per frame (and of the cfg4 row operator per launch)
    from the newest committed ncu --set full capture (profiles/*/traffic.json)."""
    for p in sorted(ROOT.glob("profiles/*/traffic.json"), reverse=True):
        try:
            return json.loads(p.read_text())
        except (OSError, ValueError):
            continue
    return None


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
        return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,power.draw.instant,power.limit")

    def __init__(self, index: int):
        self.index, self.proc, self.path = index, None, None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
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
        rows = [p for p in ([q.strip() for q in ln.split(",")] for ln in Path(self.path).read_text().splitlines())
                if len(p) == 8 and p[0].isdigit()]
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[2 + i].lower() == "active"})
        def num(v):
            try:
                return float(v)
            except ValueError:
                return None
        power = [x for x in (num(r[6]) for r in rows) if x is not None]
        return {"sm_mhz": statistics.median(int(r[0]) for r in rows), "sm_max_mhz": int(rows[0][1]),
                "reasons": reasons, "samples": len(rows),
                # board power over the same window (the steady state is power-limited when it sits at the limit)
                "power_w": statistics.median(power) if power else None, "power_limit_w": num(rows[0][7])}


def grid(cfg):
    return np.linspace(*cfg["x"], cfg["nx"]), np.linspace(*cfg["z"], cfg["nz"])


def frame_scatterers(cfg, frames, seed=2025):
    """Seeded per-frame speckle: frame f uses default_rng(seed + f) (global index)."""
    sx = np.empty((len(frames), cfg["n_scat"]))
    sz, a = np.empty_like(sx), np.empty_like(sx)
    for k, f in enumerate(frames):
        rng = np.random.default_rng(seed + int(f))
        sx[k] = rng.uniform(*cfg["region_x"], cfg["n_scat"])
        sz[k] = rng.uniform(*cfg["region_z"], cfg["n_scat"])
        a[k] = rng.standard_normal(cfg["n_scat"])
    return sx, sz, a


# ------------------------------------------------------------ CPU baselines


def cpu_baseline(budget_pixels: int, workers=None, target_s: float = 0.0):
    """Reference DAS algorithm (oracle port) on a bounded pixel sample of one cfg2 frame.

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


def cfg1_line_setup():
    """The cfg1 anchor line of SURVEY §8(c): 64 el, 0.3 mm, 5 MHz, 20 MHz, focused
    Tx FixedCount(64) at 20 mm, FNumber(1.5), RF zero-padded to 2048, 256 depths
    5-40 mm, x = 0; theta and epsilon from the reference (tests/golden)."""
    from oracle import geom, tidas as ot
    g = np.load(ROOT / "tests/golden/ref_vectors.npz")
    n_el, pitch, fs, c, f0 = 64, 0.3e-3, 20e6, 1540.0, 5e6
    traces, tx_xs = ot.reference_frame(20e-3, 20e-3, n_el=n_el, pitch=pitch, fs=fs, c=c, f0=f0, fbw=0.6,
                                       tx_half=32)
    padded = np.zeros((n_el, 2048))
    padded[:, :traces.shape[1]] = traces
    half = geom.ref_aperture_half(20e-3, ("fnumber", 1.5), n_el, pitch, c / f0)
    idx = np.arange(-half, half)
    delays = geom.receive_delays(0.0, 20e-3, (idx + 0.5) * pitch, c)
    depths = np.linspace(5e-3, 40e-3, 256)
    t_stars = geom.focused_expected_arrival(0.0, depths, 20e-3, tx_xs, c)
    return dict(traces=padded, fs=fs, idx=idx, delays=delays, thetas=g["C1_theta"], t_stars=t_stars,
                eps=float(g["C1_eps"]), depths=depths, n_el=n_el, pitch=pitch, c=c, f0=f0)


def tidas_line_cpu_baseline(trials: int = 5):
    """Reference-native tidas_line (tidas.py:493-531, oracle restatement), one
    process, median of ``trials`` timed runs after one warm-up — the harness of
    experiments.py:440-447."""
    from oracle import tidas as ot
    s = cfg1_line_setup()
    run = lambda: ot.tidas_line(s["traces"], s["fs"], 0.0, s["idx"], s["delays"], s["thetas"],  # noqa: E731
                                s["t_stars"], s["eps"])
    run()
    ts = []
    for _ in range(trials):
        t0 = time.perf_counter()
        run()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts)


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
            "data": DATA, "config": workload_config(args.frames, args.gpus),
            "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": workers, "kind": "port",
                             "sample": sample + " (oracle simulator frame rounded to float32; float64 arithmetic; "
                                                "host cores, oracle port of the reference algorithm)",
                             "cpu_model": cpu_model()},
            "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ GPU run


def nccl_env():
    """Keep NCCL's communicator log (read at communicator creation). An
    NCCL_DEBUG already in the environment (the launcher's own choice of level
    and destination) is left exactly as it is."""
    if "NCCL_DEBUG" in os.environ:
        return
    log_dir = ROOT / "gpurun_out" if (ROOT / "gpurun_out").is_dir() else Path(tempfile.gettempdir())
    os.environ["NCCL_DEBUG"] = "INFO"
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT,GRAPH,NVLS")
    os.environ.setdefault("NCCL_DEBUG_FILE", str(log_dir / "nccl_bench.%h.%p.log"))


def nccl_summary():
    """Transport facts from this process's NCCL log (P2P / NVLink / NVLS)."""
    path = os.environ.get("NCCL_DEBUG_FILE", "")
    if not path:  # the environment's own NCCL_DEBUG setting: its output goes to stderr
        return {"log": None, "NCCL_DEBUG": os.environ.get("NCCL_DEBUG")}
    p = Path(path.replace("%h", platform.node()).replace("%p", str(os.getpid())))
    if not p.exists():  # NCCL expands %h itself: look for this process's file under any host name
        hits = sorted(p.parent.glob(Path(path).name.replace("%h", "*").replace("%p", str(os.getpid()))))
        if not hits:
            return {"log": str(p), "found": False, "NCCL_DEBUG": os.environ.get("NCCL_DEBUG")}
        p = hits[0]
    text = p.read_text(errors="replace")
    return {"log": str(p), "found": True, "nvls": "NVLS" in text and "NVLS multicast support is not available" not in text,
            "p2p": "via P2P" in text, "lines": text.count("\n")}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--frames", type=int, default=256, help="cfg2 frames per GPU per step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-tidas", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the cfg1 / cfg3 / cfg5 DAS lines")
    ap.add_argument("--cpu-pixels", type=int, default=0, help="cpu_baseline pixel sample (0 = auto)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    from paper_2507_15464_b200 import parallel
    if parallel.needs_relaunch(args.gpus):
        nccl_env()
        return parallel.relaunch(args.gpus, str(Path(__file__).resolve()), sys.argv[1:])
    nccl_env()

    import torch
    import torch.distributed as dist
    import paper_2507_15464_b200 as tb
    from paper_2507_15464_b200 import imaging

    rank, world = parallel.init()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but the launcher started {world} rank(s)")
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if args.warmup < 3:
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)
    stream = torch.cuda.current_stream()

    dist_on = world > 1 or parallel.rehearsal()  # rehearsal: one rank, every collective issued

    def barrier():
        if dist_on:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v):
        if dist_on:
            t = torch.tensor([v], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return float(t.item())
        return v

    def timed(fn, steps, warmup):
        """ms per call: barrier + sync, CUDA events on the launch stream, max over ranks."""
        for _ in range(warmup):
            fn()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            fn()
        e1.record(stream)
        barrier()
        return max_over_ranks(e0.elapsed_time(e1)) / steps

    aux_errors = {}

    def aux_failed(section, exc):
        """The sections after the headline (row operator, sweep, other configs, CPU
        baselines) are reported beside it; one that raises is recorded in the line's
        ``aux_errors`` and the headline still prints. A rank that fails alone leaves
        its peers in a collective: the process group's timeout then ends the run."""
        aux_errors[section] = f"{type(exc).__name__}: {exc}"[:400]
        print(f"warning: bench section {section!r} failed: {aux_errors[section]}", file=sys.stderr, flush=True)

    hbm, peak_kind = peaks()

    # ---------------------------------------------------- cfg2 headline
    cfg = CFG2
    F = args.frames
    total_frames = F * world
    fa, fb = parallel.shard_range(total_frames, rank, world)
    frames = list(range(fa, fb))
    x, z = grid(cfg)
    sx, sz, amp = frame_scatterers(cfg, frames)
    synth_kw = {k: cfg[k] for k in ("n_el", "pitch", "fs", "c", "f0", "fbw", "n_samples")}
    rf = tb.synthesize_batch(sx, sz, amp, angles=[0.0], dtype=torch.float32, device=dev, **synth_kw)
    plan = tb.plane_wave_plan(n_el=cfg["n_el"], pitch=cfg["pitch"], fs=cfg["fs"], c=cfg["c"],
                              n_samples=cfg["n_samples"], x=x, z=z, angles=[0.0], f_number=cfg["f_number"],
                              device=dev)
    ws = imaging.DasWorkspace(plan, dev)
    img = torch.empty((len(frames), cfg["nz"], cfg["nx"]), device=dev)
    per_launch = min(len(frames), ws.chunk)

    def step():
        # frames are independent: every rank images its own shard, no collective
        tb.das_image(rf, plan, out=img, workspace=ws)

    for _ in range(args.warmup):
        step()

    # the same step, untimed, around the timed region keeps the GPU under its
    # load long enough for nvidia-smi's 100 ms samples; the step count is agreed
    # over the ranks (every rank must issue the same collectives)
    barrier()
    t0 = time.perf_counter()
    for _ in range(3):
        step()
    barrier()
    per_step = max_over_ranks((time.perf_counter() - t0) / 3)
    n_pre, n_post = max(1, int(0.6 / per_step)), max(1, int(0.4 / per_step))
    with Clocks(local) as clk:
        for _ in range(n_pre):
            step()
        ms_step = timed(step, args.steps, 0)
        for _ in range(n_post):
            step()
        torch.cuda.synchronize()
    clocks = clk.summary()
    clocks["window"] = "sampled every 100 ms over 0.6 s of the same step, the timed steps, and 0.4 s more"
    value = total_frames / (ms_step / 1e3)
    n_launch = -(-len(frames) // per_launch)
    launches = args.steps * n_launch * 2

    # K1 / K2 separately, on the per-launch frame count of the step
    # (back-to-back pairs with no host sync in between, so the clocks stay at the step's)
    an = ws.buf[:per_launch]
    evs = []
    for _ in range(8):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ev[0].record(stream)
        tb.rf_analytic(rf[:per_launch], plan.prec, out=an, sample_range=plan.sample_range())  # as das_image
        ev[1].record(stream)
        tb.das_from_analytic(an, plan, out=img[:per_launch])
        ev[2].record(stream)
        evs.append(ev)
    torch.cuda.synchronize()
    k1_ms = [ev[0].elapsed_time(ev[1]) / per_launch for ev in evs[2:]]
    k2_ms = [ev[1].elapsed_time(ev[2]) / per_launch for ev in evs[2:]]
    k1, k2 = statistics.median(k1_ms), statistics.median(k2_ms)
    pipe_gbs = BYTES_PER_FRAME_CFG2 / ((k1 + k2) / 1e3) / 1e9
    tr = committed_traffic()
    roofline = {
        "bound": "hbm", "achieved": pipe_gbs, "peak": hbm, "unit": "GB/s", "frac": pipe_gbs / hbm,
        "traffic": tr["das_pipeline_bytes_per_frame"] * per_launch if tr else None,
        "traffic_source": tr.get("source") if tr else None,
        "kernel": f"das pipeline per launch of {per_launch} frames: tidas_rf_analytic (K1) + das_image_kernel (K2)",
        "bytes_per_launch": BYTES_PER_FRAME_CFG2 * per_launch, "frames_per_launch": per_launch,
        "peak_source": peak_kind, "per_frame_us": {"K1_analytic": k1 * 1e3, "K2_das": k2 * 1e3},
        "step_frac": BYTES_PER_FRAME_CFG2 * value / world / 1e9 / hbm}
    pairs = k2_live_pairs(cfg, x, z)
    smem_peak = 148 * 128 * (clocks.get("sm_mhz") or 1965) * 1e6 / 1e9  # GB/s, 128 B/clk/SM
    smem_ach = pairs * 24 / (k2 * 1e-3) / 1e9
    k2_smem = {"bound": "smem", "achieved": smem_ach, "peak": smem_peak, "unit": "GB/s", "frac": smem_ach / smem_peak,
               "live_pairs_per_frame": pairs, "bytes_per_pair": 24, "kernel": "das_image_kernel (K2)",
               "note": "shared-memory gather roofline of K2 (128 B/clk/SM at the measured SM clock); "
                       "the HBM roofline above is the contract metric"}
    # the HBM fraction this pipeline could reach at both kernels' own floors: K1 at HBM
    # speed on its RF read + complex64 write, K2 at the shared-memory gather floor
    r_lo, r_hi = plan.sample_range()  # K1 stores only the samples K2's taps can read
    k1_floor_us = 128 * (4096 * 4 + (r_hi - r_lo + 1) * 8) / (hbm * 1e9) * 1e6
    k2_floor_us = pairs * 24 / (smem_peak * 1e9) * 1e6
    roofline["ceiling"] = {
        "frac": BYTES_PER_FRAME_CFG2 / ((k1_floor_us + k2_floor_us) * 1e-6) / 1e9 / hbm,
        "K1_floor_us": k1_floor_us, "K2_floor_us": k2_floor_us,
        "note": "HBM fraction at K1's HBM floor (RF in + the stored complex64 sample range out) plus K2's shared-memory "
                "gather floor (24 B per live pixel-channel pair at 128 B/clk/SM): the DAS gather, not HBM, "
                "bounds the pipeline; achieved / ceiling = frac / ceiling.frac"}

    # the same step at an L2-sized chunk: the analytic intermediate of 24 frames
    # (~53 MB) stays in L2 between K1 and K2 and is overwritten there by the next
    # chunk, at the price of shorter launches (more last-wave tails)
    plan_l2 = tb.plane_wave_plan(n_el=cfg["n_el"], pitch=cfg["pitch"], fs=cfg["fs"], c=cfg["c"],
                                 n_samples=cfg["n_samples"], x=x, z=z, angles=[0.0], f_number=cfg["f_number"],
                                 device=dev)
    plan_l2.chunk_bytes = 24 * cfg["n_el"] * cfg["n_samples"] * 8
    ws_l2 = imaging.DasWorkspace(plan_l2, dev)
    ms_l2 = timed(lambda: tb.das_image(rf, plan_l2, out=img, workspace=ws_l2), max(3, args.steps // 2), 2)
    tr_l2 = (tr or {}).get("l2_chunk")
    roofline["l2_resident_chunk"] = {
        "chunk_frames": ws_l2.chunk, "frames_per_s": total_frames / (ms_l2 / 1e3),
        "dram_bytes_per_frame": tr_l2.get("dram_bytes_per_frame") if tr_l2 else None,
        "x_algorithmic": tr_l2.get("x_algorithmic") if tr_l2 else None,
        "traffic_source": tr_l2.get("source") if tr_l2 else None,
        "note": "DasPlan.chunk_bytes sized for L2: DRAM traffic near the algorithmic bytes, lower throughput; "
                "the default chunk (headline) is the faster one"}
    del ws_l2, plan_l2

    # e2e through the public API with pinned host buffers (HostPipeline: H2D of
    # chunk i+1 || K1 + K2 of chunk i || D2H of chunk i-1, three streams)
    host_rf = torch.empty(rf.shape, dtype=torch.float32, pin_memory=True)
    host_rf.copy_(rf)
    host_img = torch.empty(img.shape, dtype=torch.float32, pin_memory=True)
    pipe = tb.HostPipeline(plan, chunk=16)
    for _ in range(max(1, min(args.warmup, 3))):
        pipe.run(host_rf, host_img)
    pipe.synchronize()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    pipe.wait_for(stream)
    for _ in range(args.steps):
        pipe.run(host_rf, host_img)
    pipe.join(stream)
    e1.record(stream)
    barrier()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1)) / args.steps
    rf_dev = torch.empty_like(rf)
    h2d_ms = timed(lambda: rf_dev.copy_(host_rf, non_blocking=True), 5, 1)
    h2d_gbs = host_rf.numel() * 4 / h2d_ms / 1e6
    e2e = {"value": total_frames / (e2e_ms / 1e3), "unit": "frames/s",
           "h2d_bytes_per_step": int(host_rf.numel() * 4), "d2h_bytes_per_step": int(host_img.numel() * 4),
           "ms_per_step": e2e_ms, "api": "HostPipeline.run (pinned host RF -> pinned host images), chunk 16",
           "bound": {"kind": "pcie_h2d", "h2d_GBps_measured": h2d_gbs,
                     "frac": host_rf.numel() * 4 / (e2e_ms / 1e3) / 1e9 / h2d_gbs}}
    launches_e2e = args.steps * pipe.launches(len(frames))
    del rf_dev, host_rf, host_img, pipe

    # ------------------------------------------------ tiDAS row operator
    tidas = None
    try:
        if not args.no_tidas:
            dx = x[1] - x[0]
            pkw = dict(n_el=cfg["n_el"], pitch=cfg["pitch"], fs=cfg["fs"], c=cfg["c"], f0=cfg["f0"], fbw=cfg["fbw"],
                       f_number=cfg["f_number"], n_samples=cfg["n_samples"])
            K2d, _ = tb.build_row_kernels(z, 129, dx, neighbourhood=8, **pkw)
            gen = torch.Generator(device=dev).manual_seed(7 + rank)
            M2 = 512  # cfg2 maps per GPU per step: 256 MiB in + 256 MiB out, larger than L2
            maps2 = (torch.rand((M2, cfg["nz"], cfg["nx"]), device=dev, generator=gen) < 0.02).float() * \
                torch.randn((M2, cfg["nz"], cfg["nx"]), device=dev, generator=gen)
            out2 = torch.empty_like(maps2)
            t2 = timed(lambda: tb.tidas_rowconv(maps2, K2d, out=out2), args.steps, args.warmup)
            g2 = (BYTES_PER_MAP_CFG2 * M2 + K2d.numel() * 4) / (t2 / 1e3) / 1e9
            del maps2, out2
            # cfg4: K [2048][129] built by K5 on the cfg4 grid, 256 maps sharded over the ranks
            c4 = CFG4
            x4, z4 = np.linspace(*c4["x"], c4["nx"]), np.linspace(*c4["z"], c4["nz"])
            k5_ms = timed(lambda: tb.build_row_kernels(z4, c4["taps"], x4[1] - x4[0],
                                                       neighbourhood=c4["neighbourhood"], **pkw), 3, 1)
            K4, th4 = tb.build_row_kernels(z4, c4["taps"], x4[1] - x4[0], neighbourhood=c4["neighbourhood"], **pkw)
            m0, m1 = parallel.shard_range(c4["maps"], rank, world)
            M = m1 - m0
            gen4 = torch.Generator(device=dev).manual_seed(40 + rank)
            maps4 = (torch.rand((M, c4["nz"], c4["nx"]), device=dev, generator=gen4) < c4["density"]).float() * \
                torch.randn((M, c4["nz"], c4["nx"]), device=dev, generator=gen4)
            y4, a4 = torch.empty_like(maps4), torch.empty_like(maps4)
            tf = timed(lambda: tb.tidas_rowconv(maps4, K4, out=y4), max(3, min(args.steps, 10)), 2)
            ta = timed(lambda: tb.tidas_rowconv_adjoint(y4, K4, out=a4), max(3, min(args.steps, 10)), 2)
            # adjoint identity <A x, y> = <x, A^T y> on this rank's maps (y = A x)
            lhs = float((y4.double() * y4.double()).sum())
            rhs = float((maps4.double() * a4.double()).sum())
            g4 = (BYTES_PER_MAP_CFG4 * M + K4.numel() * 4) / (tf / 1e3) / 1e9
            ga = (BYTES_PER_MAP_CFG4 * M + K4.numel() * 4) / (ta / 1e3) / 1e9
            cpu_rowconv = None
            if rank == 0 and world == 1 and not args.no_cpu_baseline:
                # the row operator's float64 CPU restatement (no reference counterpart,
                # SURVEY §8(d)), one process, on a bounded sample of one cfg4 map
                from oracle import tidas as ot
                rows = 128
                g1 = maps4[0, :rows].double().cpu().numpy()[None]
                t0 = time.perf_counter()
                ot.rowconv_fwd(g1, K4[:rows].double().cpu().numpy())
                ct = time.perf_counter() - t0
                cpu_rowconv = {"kind": "port (restatement)", "cores": 1, "unit": "maps/s (fwd)",
                               "value": rows / c4["nz"] / ct, "sample": f"{rows} of {c4['nz']} rows of one cfg4 map",
                               "cpu_model": cpu_model()}
            tidas = {
                "cfg2_fwd": {"value": M2 * world / (t2 / 1e3), "unit": "maps/s", "maps_per_step_per_gpu": M2,
                             "ms_per_step": t2, "scaling": "weak",
                             "roofline": {"bound": "hbm", "achieved": g2, "peak": hbm, "unit": "GB/s", "frac": g2 / hbm,
                                          "traffic": None, "kernel": "rowconv_tc1_kernel<fwd> (tcgen05 3xTF32)"}},
                "cfg4_fwd_adj": {"value": c4["maps"] / ((tf + ta) / 1e3), "unit": "maps/s (fwd+adj)", "fwd_ms": tf,
                                 "adj_ms": ta, "maps_per_gpu": M, "maps_total": c4["maps"], "scaling": "strong",
                                 "adjoint_identity_rel": abs(lhs - rhs) / max(abs(lhs), 1e-300),
                                 "roofline": {"bound": "hbm", "achieved": g4, "peak": hbm, "unit": "GB/s",
                                              "frac": g4 / hbm, "adj_frac": ga / hbm,
                                              "traffic": (tr or {}).get("rowconv_cfg4_bytes_per_launch"),
                                              "kernel": f"rowconv_tc1_kernel<fwd> (tcgen05 3xTF32), {M} maps/launch"}},
                "row_kernels_k5": {"rows": c4["nz"], "taps": c4["taps"], "ms": k5_ms, "api": "build_row_kernels "
                                   "(tidas_build_row_kernels: FP64 PSF per depth row + LS theta)",
                                   "theta_range": [float(th4.min()), float(th4.max())]},
                "cpu_baseline": cpu_rowconv,
            }
            del maps4, y4, a4
            torch.cuda.empty_cache()
            # cfg5 ("run DAS and tiDAS at 1/2/4/8 GPUs with frame sharding"): K5 on the cfg5 array, 1024 maps sharded
            c5 = CFG5T
            x5, z5 = np.linspace(*c5["x"], c5["nx"]), np.linspace(*c5["z"], c5["nz"])
            K5k, th5 = tb.build_row_kernels(z5, c5["taps"], x5[1] - x5[0], neighbourhood=c5["neighbourhood"],
                                            **c5["probe"])
            m0, m1 = parallel.shard_range(c5["maps"], rank, world)
            M5 = m1 - m0
            gen5 = torch.Generator(device=dev).manual_seed(50 + rank)
            maps5 = (torch.rand((M5, c5["nz"], c5["nx"]), device=dev, generator=gen5) < c5["density"]).float() * \
                torch.randn((M5, c5["nz"], c5["nx"]), device=dev, generator=gen5)
            y5, a5 = torch.empty_like(maps5), torch.empty_like(maps5)
            tf5 = timed(lambda: tb.tidas_rowconv(maps5, K5k, out=y5), max(3, min(args.steps, 10)), 2)
            ta5 = timed(lambda: tb.tidas_rowconv_adjoint(y5, K5k, out=a5), max(3, min(args.steps, 10)), 2)
            lhs5 = float((y5.double() * y5.double()).sum())
            rhs5 = float((maps5.double() * a5.double()).sum())
            g5 = (BYTES_PER_MAP_CFG5 * M5 + K5k.numel() * 4) / (tf5 / 1e3) / 1e9
            ga5 = (BYTES_PER_MAP_CFG5 * M5 + K5k.numel() * 4) / (ta5 / 1e3) / 1e9
            tidas["cfg5_fwd_adj"] = {
                "value": c5["maps"] / ((tf5 + ta5) / 1e3), "unit": "maps/s (fwd+adj)", "fwd_ms": tf5, "adj_ms": ta5,
                "fwd_maps_per_s": c5["maps"] / (tf5 / 1e3), "maps_per_gpu": M5, "maps_total": c5["maps"],
                "scaling": "strong", "adjoint_identity_rel": abs(lhs5 - rhs5) / max(abs(lhs5), 1e-300),
                "kernels": "K5 on the cfg5 array and grid (1024 rows x 129 taps), theta in "
                           f"[{float(th5.min()):.4f}, {float(th5.max()):.4f}]",
                "roofline": {"bound": "hbm", "achieved": g5, "peak": hbm, "unit": "GB/s", "frac": g5 / hbm,
                             "adj_frac": ga5 / hbm, "traffic": None,
                             "kernel": f"rowconv_tc1_kernel<fwd> (tcgen05 3xTF32), {M5} maps/launch"}}
            del maps5, y5, a5
            torch.cuda.empty_cache()
    except Exception as e:  # noqa: BLE001 — an auxiliary section never costs the headline line
        aux_failed('tidas', e)

    # ---------------- the paper's 600 x 600 theta / error sweep
    sweep = None
    try:
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
                     "finite_cells": int(np.isfinite(th600).sum()), "paper_cpu_minutes": {"das": 28.35, "tidas": 21.11},
                     "api": "error_sweep (theta, local and global error matrices of run_error_sweep), "
                            "600 scatterer depths x 600 reference profiles, 5-42 mm, 7 MHz, Tx focus 25 mm",
                     "timing": "CUDA events around the public call (host geometry + D2H of the matrices inside)"}
            if world == 1 and not args.no_cpu_baseline:
                from oracle import theta as oth
                probe = dict(n_el=192, pitch=0.2e-3, f0=7e6, fs=50e6, c=1540.0, fbw=0.75)
                d12 = d600[::50]
                t0 = time.perf_counter()
                oth.error_sweep(d12, d12, probe, tx_focus=25e-3, half_width=eps)
                ct = time.perf_counter() - t0
                sweep["cpu_baseline"] = {"kind": "port", "cores": 1, "sample": f"{len(d12)} x {len(d12)} cells",
                                         "seconds_per_cell": ct / len(d12) ** 2,
                                         "extrapolated_600x600_minutes": ct / len(d12) ** 2 * 360000 / 60}
    except Exception as e:  # noqa: BLE001 — an auxiliary section never costs the headline line
        aux_failed('theta_error_sweep', e)

    # ------------ the other BASELINE.json DAS configs (cfg1 weak; cfg3 / cfg5 sharded, cfg3 gathered)
    others = None
    try:
        if not args.no_configs:
            sys.path.insert(0, str(ROOT / "tools"))
            import bench_configs
            res = bench_configs.run_configs(["cfg1", "cfg3", "cfg5"], rank=rank, world=world, timed=timed, hbm=hbm)
            others = {k: {q: v[q] for q in ("frames_per_s", "ms_per_step", "frames_total", "frames_per_rank",
                                             "hbm_frac", "bytes_per_frame", "rf_dtype", "transmits", "grid", "out",
                                             "scaling", "gather", "nccl_gather_frames_per_s")}
                      for k, v in res.items()}
            others["note"] = ("das_image (K1 + K2) with the RF resident in HBM, CUDA events, max over ranks; cfg3 / "
                              "cfg5 shard a fixed batch (64 / 1024 frames) over the ranks; cfg3 all-gathers its "
                              "compounded images over NCCL inside the step")
    except Exception as e:  # noqa: BLE001 — an auxiliary section never costs the headline line
        aux_failed('other_configs', e)

    # ------------------------------------------------- CPU baselines (N = 1)
    cpu = None
    line_cpu = None
    try:
        if rank == 0 and world == 1 and not args.no_cpu_baseline:
            workers = os.cpu_count() or 1
            n_px = args.cpu_pixels or max(workers * 48, 96)
            fps, n, dt, w = cpu_baseline(n_px, workers, target_s=0.0 if args.cpu_pixels else 8.0)
            cpu = {"value": fps, "unit": "frames/s", "cores": w, "kind": "port", "cpu_model": cpu_model(),
                   "sample": f"{n} seeded pixels of one cfg2 frame ({dt:.1f} s over {w} processes), "
                             "reference per-pixel algorithm (full-trace shifts + Hilbert), extrapolated to 131072 px/frame"}
            # reference-native tiDAS (tidas_line) on the cfg1 anchor line, CPU vs the drop-in
            sec = tidas_line_cpu_baseline()
            s = cfg1_line_setup()
            p1 = tb.ProbeConfig(element_count=64, pitch=0.3e-3, center_frequency=5e6, sampling_frequency=20e6,
                                sound_speed=1540.0, fractional_bandwidth=0.6)
            frame = tb.RfFrame(s["traces"], s["fs"], 0.0, 20e-3, tb.tx_aperture(20e-3, tb.FixedCount(64), p1))
            fixed = tb.rx_delay_profile(20e-3, tb.rx_aperture(20e-3, tb.FNumber(1.5), p1), p1)
            gl = []
            for k in range(6):
                t0 = time.perf_counter()
                tb.tidas_line(frame, fixed, s["thetas"], s["depths"], p1, window_half_width=s["eps"])
                if k:
                    gl.append(time.perf_counter() - t0)
            line_cpu = {"kind": "port", "cores": 1, "cpu_model": cpu_model(), "unit": "lines/s",
                        "value": 1.0 / sec, "seconds_per_line": sec,
                        "sample": "cfg1 anchor line (256 depths, 64 el, 20 MHz), median of 5 after warm-up "
                                  "(experiments.py:440-447 harness)",
                        "drop_in_seconds_per_line": statistics.median(gl),
                        "drop_in_note": "tidas_line drop-in (K3 + K4 on the GPU, host round trips inside)"}
    except Exception as e:  # noqa: BLE001 — an auxiliary section never costs the headline line
        aux_failed('cpu_baselines', e)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": DATA, "config": workload_config(F, world),
            "roofline": roofline, "k2_smem_roofline": k2_smem, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches, "gpu_launches_e2e": launches_e2e, "clocks": clocks,
            "tidas": tidas, "theta_error_sweep": sweep, "other_configs": others,
            "tidas_line_cpu_baseline": line_cpu,
            "nccl": nccl_summary() if dist_on else None,
        }
        if aux_errors:
            line["aux_errors"] = aux_errors
        if parallel.rehearsal():
            line["rehearsal"] = "TIDAS_DIST_REHEARSAL: one rank issuing the multi-rank step's collectives; not a scaling number"
        print(json.dumps(line), flush=True)
    if dist_on:
        try:
            dist.barrier()
            dist.destroy_process_group()
        except Exception as e:  # noqa: BLE001 — the line is out; a failed teardown is only worth a warning
            print(f"warning: process-group teardown failed: {e}", file=sys.stderr, flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
