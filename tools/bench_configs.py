"""Throughput of the DAS path at the other BASELINE.json configs.

  python tools/bench_configs.py [--steps 10] [--warmup 3] [--configs cfg1,cfg3,cfg5]

Each record: frames/s of K1 + K2 with the RF resident in HBM (CUDA events around
`das_image`, max over ranks), per-frame algorithmic bytes (RF in
its arrival dtype + FP32 image) and the HBM-roofline fraction. Inputs are
seeded synthetic frames simulated on the device (cfg5: scaled to std 1000,
rounded, clipped to int16 by the library quantiser). Called by bench.py with
its rank / world: cfg1 is weak-scaled (256 frames per rank); cfg3 (64 frames)
and cfg5 (1024 frames) shard a fixed batch over the ranks (strong scaling).
cfg3 all-gathers its compounded images over NCCL inside the timed step (north
star (e), BASELINE.json cfg3); cfg1 / cfg5 frames stay on their rank (no
data-path collective).
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
from paper_2507_15464_b200 import imaging, parallel  # noqa: E402

CFGS = {
    "cfg1": dict(n_el=64, pitch=0.3e-3, f0=5e6, fs=20e6, fbw=0.6, N=2048, nz=256, nx=128, z=(5e-3, 40e-3),
                 x=(-9.6e-3, 9.6e-3), angles=[0.0], frames=256, per_rank=True, n_scat=1, dtype=torch.float64,
                 out="envelope", bytes=64 * 2048 * 8 + 256 * 128 * 4, region=None),
    "cfg3": dict(n_el=128, pitch=0.3e-3, f0=5e6, fs=40e6, fbw=0.6, N=4096, nz=1024, nx=512, z=(5e-3, 45e-3),
                 x=(-19.2e-3, 19.2e-3), angles=list(np.deg2rad(np.linspace(-10, 10, 11))), frames=64,
                 per_rank=False, gather=True, n_scat=2000, n_bright=5, dtype=torch.float32, out="coherent",
                 bytes=11 * 128 * 4096 * 4 + 1024 * 512 * 4, region=((-20e-3, 20e-3), (5e-3, 45e-3))),
    "cfg5": dict(n_el=192, pitch=0.3e-3, f0=5e6, fs=40e6, fbw=0.6, N=8192, nz=1024, nx=1024, z=(5e-3, 60e-3),
                 x=(-28.8e-3, 28.8e-3), angles=[0.0], frames=1024, per_rank=False, n_scat=4000, dtype=torch.int16,
                 out="envelope", bytes=192 * 8192 * 2 + 1024 * 1024 * 4, region=((-28.8e-3, 28.8e-3), (5e-3, 60e-3))),
}


def make_rf(name, c, frames):
    """Seeded frames: global frame f draws from default_rng(7000 + f) (shard-invariant)."""
    F = len(frames)
    if name == "cfg1":  # single point scatterer (0, 20 mm), replicated frames
        sx, sz, a = np.zeros((F, 1)), np.full((F, 1), 20e-3), np.ones((F, 1))
    else:
        (x0, x1), (z0, z1) = c["region"]
        S = c["n_scat"] + c.get("n_bright", 0)
        sx, sz, a = np.empty((F, S)), np.empty((F, S)), np.empty((F, S))
        for k, f in enumerate(frames):
            rng = np.random.default_rng(7000 + f)
            sx[k], sz[k], a[k] = rng.uniform(x0, x1, S), rng.uniform(z0, z1, S), rng.standard_normal(S)
            if c.get("n_bright"):
                a[k, c["n_scat"]:] = 20.0  # bright point targets
    # cfg5: simulated in float32, each frame scaled to std 1000, rounded, clipped (library quantiser)
    return tb.synthesize_batch(sx, sz, a, angles=c["angles"], n_el=c["n_el"], pitch=c["pitch"], fs=c["fs"],
                               c=1540.0, f0=c["f0"], fbw=c["fbw"], n_samples=c["N"], dtype=c["dtype"],
                               target_std=1000.0)


def _default_timed(fn, steps, warmup):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def run_configs(names, steps=10, warmup=3, echo=False, rank=0, world=1, timed=None, hbm=None):
    """Frames/s of das_image (K1 + K2, RF resident) per config; returns {name: record}."""
    timed = timed or _default_timed
    if hbm is None:
        p = ROOT / "MEASURED_PEAKS.json"
        hbm = json.loads(p.read_text())["hbm_gbs"] if p.exists() else 6650.0
    res = {}
    for name in names:
        c = CFGS[name]
        total = c["frames"] * (world if c["per_rank"] else 1)
        f0, f1 = parallel.shard_range(total, rank, world)
        rf = make_rf(name, c, list(range(f0, f1)))
        x, z = np.linspace(*c["x"], c["nx"]), np.linspace(*c["z"], c["nz"])
        plan = tb.plane_wave_plan(n_el=c["n_el"], pitch=c["pitch"], fs=c["fs"], c=1540.0, n_samples=c["N"],
                                  x=x, z=z, angles=c["angles"], f_number=1.5, out=c["out"])
        ws = imaging.DasWorkspace(plan)
        img = torch.empty((rf.shape[0], c["nz"], c["nx"]), device="cuda")
        gather = (world > 1 or parallel.rehearsal()) and c.get("gather", False)
        full = torch.empty((total, c["nz"], c["nx"]), device="cuda") if gather else None
        n_local = int(rf.shape[0])
        # sub-chunks of whole 8-frame groups (K2's frames per thread); with two or
        # more, the all-gather of one overlaps the DAS of the next
        sub = max(8, (n_local // 2) // 8 * 8)
        pipelined = gather and total % world == 0 and n_local >= 2 * sub

        def step():
            if pipelined:  # NCCL over NVLink, chunk-major order (parallel.chunk_major_index)
                parallel.pipelined_gather(
                    lambda a, b: tb.das_image(rf[a:b], plan, out=img[a:b], workspace=ws), n_local, full, sub=sub,
                    layout="chunk_major")
                return
            tb.das_image(rf, plan, out=img, workspace=ws)
            if gather:  # NCCL over NVLink: every rank receives the whole batch's images
                parallel.gather_images(img, total, out=full)

        ms = timed(step, steps, warmup)
        ms_nccl, peer_err = None, None
        if gather:
            # the same gather fused into K2: the epilogue stores every pixel into each
            # peer's symmetric-memory copy over NVLink, one device barrier per step
            pg, peer_err = parallel.try_peer_gather(total, (c["nz"], c["nx"]), torch.float32, img.device)
            if pg is not None:
                def step_peer():
                    pg.begin()
                    tb.das_image(rf, plan, out=pg.local(), workspace=ws, peers=pg.peers)
                    pg.end()

                ms_peer = timed(step_peer, steps, warmup)
                if pipelined:
                    order = [parallel.chunk_major_index(f, n_local, world, sub) for f in range(total)]
                    ref = full[torch.tensor(order, device=full.device)]
                else:
                    ref = full
                # every rank must hold the NCCL result bit for bit; the ranks agree on the verdict
                # (MIN over the group) so that none reports the peer timing alone
                same = torch.tensor([int(torch.equal(pg.local(), img) and torch.equal(pg.buf, ref))],
                                    device=img.device, dtype=torch.int32)
                if world > 1:
                    torch.distributed.all_reduce(same, op=torch.distributed.ReduceOp.MIN)
                if int(same.item()):
                    ms_nccl, ms = ms, ms_peer
                else:  # keep the NCCL number and say why
                    peer_err = "peer-gathered images differ from the NCCL all-gather on at least one rank"
                del pg
        fps = total / (ms / 1e3)
        gbs = c["bytes"] * fps / world / 1e9
        res[name] = {"frames_total": total, "frames_per_rank": int(rf.shape[0]), "ms_per_step": ms,
                     "frames_per_s": fps, "bytes_per_frame": c["bytes"], "hbm_GBps_per_gpu": gbs,
                     "hbm_frac": gbs / hbm, "rf_dtype": str(c["dtype"]).replace("torch.", ""),
                     "transmits": len(c["angles"]), "grid": [c["nz"], c["nx"]], "out": c["out"],
                     "chunk_frames": ws.chunk, "scaling": "weak" if c["per_rank"] else "strong",
                     "gather": ("K2 epilogue stores into every peer's symmetric-memory image buffer over "
                                "NVLink (tidas_das_image_peers) + device barrier; NCCL all-gather timed beside it"
                                if ms_nccl is not None else
                                ("NCCL all_gather_into_tensor of the images, pipelined per "
                                 f"{sub} frames" if pipelined else "NCCL all_gather_into_tensor of the images")
                                + (f" (peer stores not used: {peer_err})" if peer_err else ""))
                               if gather else "none",
                     "nccl_gather_frames_per_s": total / (ms_nccl / 1e3) if ms_nccl else None,
                     "checksum": float(img.double().sum())}
        if echo:
            print(json.dumps({name: res[name]}), flush=True)
        del rf, img, ws, full
        torch.cuda.empty_cache()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--configs", default="cfg1,cfg3,cfg5")
    ap.add_argument("--lib", default=None, help="a variant libtidas_b200.so (tools/build_variant.sh)")
    args = ap.parse_args()
    if args.lib:
        from paper_2507_15464_b200 import _lib
        _lib.load(Path(args.lib))
    print(json.dumps(run_configs(args.configs.split(","), args.steps, args.warmup, echo=True)))


if __name__ == "__main__":
    main()
