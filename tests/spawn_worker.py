"""Launch-path stand-in for bench.py (CPU, gloo): ``python tests/spawn_worker.py N``
re-launches itself as N ranks through parallel.relaunch exactly like
``bench.py --gpus N`` does, checks WORLD_SIZE, shards seeded "frames", gathers
them with the bench's pipelined all-gather and the cfg3 / cfg5 padded gather,
and rank 0 prints one JSON line."""
import json
import sys
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2507_15464_b200 import parallel  # noqa: E402


def frame_image(f: int) -> torch.Tensor:
    return torch.full((2, 3), float(f)) + torch.arange(6.0).view(2, 3) / 10


def main() -> int:
    n = int(sys.argv[1])
    if parallel.needs_relaunch(n):
        return parallel.relaunch(n, str(Path(__file__).resolve()), sys.argv[1:])
    rank, world = parallel.init("gloo")
    if world != n:
        raise SystemExit(f"asked for {n} ranks, launcher started {world}")
    per_rank = 5                                   # weak (cfg2): same frames per rank
    a, b = parallel.shard_range(per_rank * world, rank, world)
    local = torch.stack([frame_image(f) for f in range(a, b)])
    out = torch.empty((per_rank * world, 2, 3))
    parallel.pipelined_gather(lambda c0, c1: local[c0:c1], b - a, out, sub=2)
    # the bench's zero-copy chunk-major layout
    out_cm = torch.empty((per_rank * world, 2, 3))
    parallel.pipelined_gather(lambda c0, c1: local[c0:c1], b - a, out_cm, sub=2, layout="chunk_major")
    cm_ok = all(torch.equal(out_cm[parallel.chunk_major_index(f, per_rank, world, 2)], frame_image(f))
                for f in range(per_rank * world))
    fixed = 7                                      # strong (cfg3 / cfg5): fixed batch, ragged shards
    c0, c1 = parallel.shard_range(fixed, rank, world)
    loc2 = torch.stack([frame_image(f) for f in range(c0, c1)])
    full = parallel.gather_images(loc2, fixed)
    ok = bool(cm_ok and torch.equal(out, torch.stack([frame_image(f) for f in range(per_rank * world)])) and
              torch.equal(full, torch.stack([frame_image(f) for f in range(fixed)])))
    oks = [None] * world
    dist.all_gather_object(oks, ok)
    if rank == 0:
        print(json.dumps({"world": world, "ok": all(oks), "collectives": parallel.collectives_on()}), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
