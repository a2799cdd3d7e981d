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
    q.put((rank, full.numpy().tolist()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n_units", [7, 8])
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
