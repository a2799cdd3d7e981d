"""Frame sharding + image gather over a real 2-process gloo group (CPU)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2507_15464_b200.parallel import gather_images, shard_range


def test_shard_range_partitions():
    for n in (0, 1, 7, 64, 1024):
        for w in (1, 2, 3, 8):
            spans = [shard_range(n, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n_units, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a, b = shard_range(n_units, rank, world)
    # per-frame "image" that depends only on the frame index (as DAS does)
    local = torch.stack([torch.full((3, 4), float(f)) + torch.arange(12.0).view(3, 4)
                         for f in range(a, b)]) if b > a else torch.zeros((0, 3, 4))
    full = gather_images(local, n_units)
    into = gather_images(local, n_units, out=torch.full((n_units, 3, 4), -1.0))  # caller-owned result
    assert torch.equal(full, into)
    q.put((rank, full.numpy().tolist()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n_units", [7, 8])  # padded (unequal shards) and direct (equal shards) paths
def test_gather_two_ranks_matches_single_process(n_units):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_units, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = torch.stack([torch.full((3, 4), float(f)) + torch.arange(12.0).view(3, 4)
                        for f in range(n_units)]).numpy().tolist()
    assert res[0] == want and res[1] == want


def _pipelined_worker(rank, world, port, n_local, sub, q, layout="rank_major"):
    from paper_2507_15464_b200.parallel import pipelined_gather
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    calls = []

    def compute(c0, c1):
        calls.append((c0, c1))
        f0 = rank * n_local
        return torch.stack([torch.full((2, 3), float(f0 + f)) for f in range(c0, c1)])

    out = torch.empty((world * n_local, 2, 3))
    pipelined_gather(compute, n_local, out, sub, layout=layout)
    q.put((rank, out.numpy().tolist(), calls))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n_local,sub", [(8, 3), (6, 6), (5, 1)])
def test_pipelined_gather_two_ranks(n_local, sub):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_pipelined_worker, args=(r, 2, port, n_local, sub, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {r: (o, c) for r, o, c in (q.get(timeout=120) for _ in procs)}
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = [[[float(f)] * 3] * 2 for f in range(2 * n_local)]
    chunks = [(c0, min(n_local, c0 + sub)) for c0 in range(0, n_local, sub)]
    for r in (0, 1):
        assert res[r][0] == want
        assert res[r][1] == chunks


@pytest.mark.parametrize("n_local,sub", [(8, 3), (6, 6), (5, 1), (7, 64)])
def test_pipelined_gather_chunk_major_two_ranks(n_local, sub):
    """The bench's zero-copy layout: each sub-chunk all-gathered straight into a
    contiguous slice of the output; chunk_major_index maps global units."""
    from paper_2507_15464_b200.parallel import chunk_major_index
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_pipelined_worker, args=(r, 2, port, n_local, sub, q, "chunk_major"))
             for r in range(2)]
    for p in procs:
        p.start()
    res = {r: (o, c) for r, o, c in (q.get(timeout=120) for _ in procs)}
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in (0, 1):
        out = res[r][0]
        assert sorted(row[0][0] for row in out) == [float(f) for f in range(2 * n_local)]
        for f in range(2 * n_local):
            assert out[chunk_major_index(f, n_local, 2, sub)][0][0] == float(f)


def test_relaunch_spawns_ranks_like_bench():
    """``bench.py --gpus N`` outside torchrun re-launches itself as N ranks
    (parallel.relaunch over torch.distributed.run, 127.0.0.1): the same path,
    on gloo, with the bench's pipelined and padded gathers."""
    import json
    import subprocess
    import sys
    from pathlib import Path
    script = Path(__file__).resolve().parent / "spawn_worker.py"
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, str(script), "2"], capture_output=True, text=True, timeout=240, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(ln) for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert lines == [{"world": 2, "ok": True, "collectives": True}]


def test_rehearsal_one_rank_issues_the_collectives():
    """TIDAS_DIST_REHEARSAL=1: one process creates the group and runs the same
    gathers through it (what the one-GPU dry run of the multi-rank bench does)."""
    import json
    import subprocess
    import sys
    from pathlib import Path
    script = Path(__file__).resolve().parent / "spawn_worker.py"
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_PORT")}
    env["TIDAS_DIST_REHEARSAL"] = "1"
    r = subprocess.run([sys.executable, str(script), "1"], capture_output=True, text=True, timeout=240, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(ln) for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert lines == [{"world": 1, "ok": True, "collectives": True}]


def test_peer_destinations_skip_self_and_offset():
    from paper_2507_15464_b200.parallel import peer_destinations
    ptrs = [1000, 5000, 9000, 13000]
    assert peer_destinations(ptrs, 1, 3, 16) == [1048, 9048, 13048]
    assert peer_destinations(ptrs[:1], 0, 0, 16) == []


def _angle_worker(rank, world, port, n_angles, q):
    from paper_2507_15464_b200.parallel import compound_angle_shards, shard_range
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = torch.Generator().manual_seed(11)
    per_angle = torch.view_as_complex(torch.randn((n_angles, 2, 5, 4, 2), generator=g, dtype=torch.float64))
    a0, a1 = shard_range(n_angles, rank, world)
    iq_local = per_angle[a0:a1].sum(0)               # what an out="iq" plan over this rank's angles returns
    img = compound_angle_shards(iq_local)
    out = torch.empty((2, 5, 4), dtype=torch.float64)
    compound_angle_shards(iq_local, out=out)
    assert torch.equal(img, out)
    q.put((rank, img.numpy().tolist(), per_angle.sum(0).abs().numpy().tolist()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n_angles", [11, 4])  # cfg3's 11 angles: shards of 6 + 5
def test_angle_sharded_compounding_two_ranks(n_angles):
    """Each rank sums its own steering angles' IQ; the all-reduced magnitude is
    the coherently compounded image of all angles on every rank."""
    import numpy as np
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_angle_worker, args=(r, 2, port, n_angles, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, img, want in res:
        np.testing.assert_allclose(np.array(img), np.array(want), rtol=1e-13, atol=0)
    assert res[0][1] == res[1][1]                    # identical on both ranks


def test_compound_angle_shards_one_process_is_the_magnitude():
    from paper_2507_15464_b200.parallel import compound_angle_shards
    iq = torch.view_as_complex(torch.randn((3, 4, 5, 2)))
    assert torch.equal(compound_angle_shards(iq), iq.abs())
    with pytest.raises(ValueError):
        compound_angle_shards(iq.real)
