"""K2 with the image gather fused into its epilogue (tidas_das_image_peers).

One GPU here: the peer destinations are ordinary device buffers (the store
instruction is the same whether the address maps local HBM or a peer GPU over
NVLink), plus torch symmetric memory at world size 1 (its mapped address as the
destination) in a subprocess. The N > 1 path is timed by bench.py's cfg3 line.
"""
import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

from tests.setups import CFG2, CFG3, grid

pytestmark = pytest.mark.gpu
tb = pytest.importorskip("paper_2507_15464_b200")
from paper_2507_15464_b200 import imaging  # noqa: E402

DEV = "cuda"


def _plan_rf(cfg, nz, nx, F, out, angles=(0.0,), seed=3):
    x, z = grid(cfg, nz, nx)
    plan = tb.plane_wave_plan(n_el=cfg["n_el"], pitch=cfg["pitch"], fs=cfg["fs"], c=cfg["c"],
                              n_samples=cfg["n_samples"], x=x, z=z, angles=list(angles), out=out)
    g = torch.Generator(device=DEV).manual_seed(seed)
    rf = torch.randn((F, len(angles), cfg["n_el"], cfg["n_samples"]), device=DEV, generator=g)
    return plan, rf


def _small_chunks(plan, chunk=8):
    ws = imaging.DasWorkspace(plan)
    ws.chunk = chunk
    ws.buf = ws.buf[:chunk]
    return ws


@pytest.mark.parametrize("out_mode,angles", [("envelope", (0.0,)), ("coherent", CFG3["angles"][:3]),
                                             ("iq", (0.0,))])
def test_peer_buffers_receive_the_image_bitwise(out_mode, angles):
    """11 frames in chunks of 8 (per-chunk peer offsets), ragged 37 x 53 grid:
    every peer buffer equals the local image, and nothing outside its frames
    is touched."""
    cfg = CFG2
    F, nz, nx = 11, 37, 53
    plan, rf = _plan_rf(cfg, nz, nx, F, out_mode, angles)
    ws = _small_chunks(plan)
    ref = tb.das_image(rf, plan, workspace=ws)
    dt = ref.dtype
    guard = 5
    peers = [torch.full((F + 2 * guard, nz, nx), 7.0, dtype=torch.float32, device=DEV).to(dt) for _ in range(3)]
    out = torch.empty_like(ref)
    tb.das_image(rf, plan, out=out, workspace=ws, peers=[p[guard].data_ptr() for p in peers])
    torch.cuda.synchronize()
    assert torch.equal(out, ref)
    sentinel = torch.tensor(7.0, device=DEV).to(dt)
    for p in peers:
        assert torch.equal(p[guard:guard + F], ref)
        assert bool((p[:guard] == sentinel).all()) and bool((p[guard + F:] == sentinel).all())


def test_peer_offsets_for_a_frame_slice():
    """A rank's frames land at its own offset of every copy (the bench's layout):
    two 'ranks' imaging frames [0, 5) and [5, 11) into two shared buffers."""
    cfg = CFG2
    F, nz, nx = 11, 24, 40
    plan, rf = _plan_rf(cfg, nz, nx, F, "envelope", seed=9)
    ref = tb.das_image(rf, plan)
    bufs = [torch.zeros((F, nz, nx), device=DEV) for _ in range(2)]
    for r, (a, b) in enumerate([(0, 5), (5, 11)]):
        other = bufs[1 - r]
        tb.das_image(rf[a:b], plan, out=bufs[r][a:b], peers=[other[a].data_ptr()])
    torch.cuda.synchronize()
    assert torch.equal(bufs[0], ref) and torch.equal(bufs[1], ref)


def test_peer_argument_validation():
    cfg = CFG2
    plan, rf = _plan_rf(cfg, 16, 16, 2, "envelope")
    with pytest.raises(ValueError):
        tb.das_image(rf, plan, peers=[rf.data_ptr()] * 8)
    with pytest.raises(ValueError):
        tb.das_image(rf, plan, peers=[0])


def test_symmetric_memory_destination_world1():
    """torch symmetric memory at world size 1: K2 stores into the mapped
    symmetric buffer through its rendezvous address (subprocess: its own
    process group)."""
    worker = Path(__file__).resolve().parent / "peer_worker.py"
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, str(worker)], capture_output=True, text=True, timeout=300, env=env)
    lines = [json.loads(ln) for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert r.returncode == 0 and lines, r.stderr[-3000:]
    res = lines[-1]
    if res.get("skip"):
        pytest.skip(f"symmetric memory unavailable here: {res['skip']}")
    assert res["ok"], res
