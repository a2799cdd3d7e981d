"""Frame sharding across GPUs (north star (e)).

Frames (and tiDAS maps) are independent units: each rank owns a
contiguous range of them, computes its images with no data-path collective,
and NCCL over NVLink is used only to gather the images. Mirrors the
reference's index-gathered, worker-count-invariant sweeps
(experiments.py:195-199; test_experiments.py:124-131).
"""
from __future__ import annotations

import os
import socket
import subprocess
import sys
from typing import Optional, Sequence, Tuple

import torch
import torch.distributed as dist


def shard_range(n_units: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous [start, stop) of ``n_units`` owned by ``rank`` (balanced +-1)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank / world size")
    base, extra = divmod(n_units, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def env_rank_world() -> Tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment (1 process if unset)."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch(n: int, script: str, argv: Sequence[str], env: Optional[dict] = None) -> int:
    """Run ``script argv`` as ``n`` ranks on this node under torch.distributed.run
    (one process per GPU, rendezvous on 127.0.0.1) and return its exit code —
    what ``bench.py --gpus N`` does when it was not started by torchrun."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", script, *argv]
    return subprocess.call(cmd, env=dict(os.environ, **(env or {})))


def needs_relaunch(requested: int) -> bool:
    """True when N > 1 ranks were asked for but this process is not one of them."""
    return requested > 1 and "WORLD_SIZE" not in os.environ


def rehearsal() -> bool:
    """TIDAS_DIST_REHEARSAL=1: a single process still creates the process group
    and issues every collective of the multi-rank step (NCCL all-gathers of one
    rank, the symmetric-memory barriers) — a one-GPU dry run of the code the
    ranks of a node execute. Timings from it say nothing about NVLink."""
    return os.environ.get("TIDAS_DIST_REHEARSAL", "") not in ("", "0")


def collectives_on(group=None) -> bool:
    """True when gathers must go through the process group (more than one rank, or a rehearsal)."""
    return dist.is_initialized() and (dist.get_world_size(group) > 1 or rehearsal())


def init(backend: Optional[str] = None) -> Tuple[int, int]:
    """Initialise the process group when launched by torchrun; returns (rank, world)."""
    rank, world, local = env_rank_world()
    if world == 1 and rehearsal():
        for k, v in (("MASTER_ADDR", "127.0.0.1"), ("MASTER_PORT", str(free_port())), ("RANK", "0"),
                     ("WORLD_SIZE", "1"), ("LOCAL_RANK", "0")):
            os.environ.setdefault(k, v)
    if (world > 1 or rehearsal()) and not dist.is_initialized():
        backend = backend or ("nccl" if torch.cuda.is_available() else "gloo")
        if backend == "nccl":
            torch.cuda.set_device(local)
            # device_id: the communicator is bound to this rank's GPU and created eagerly
            dist.init_process_group(backend=backend, device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend=backend)
    return rank, world


def gather_images(local: torch.Tensor, n_units: int, out: Optional[torch.Tensor] = None,
                  group=None) -> Optional[torch.Tensor]:
    """All-gather per-rank image shards [n_local][...] into [n_units][...] on every rank.

    Equal shards are gathered by one ``all_gather_into_tensor`` straight into
    the result; shards that differ by one unit are padded to the largest shard,
    gathered and trimmed."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if not collectives_on(group):
        return local if out is None else out.copy_(local)
    tail = tuple(local.shape[1:])
    cap = shard_range(n_units, 0, world)[1]
    if n_units % world == 0 and local.is_contiguous():
        # equal shards: NCCL writes every rank's shard straight into its slice of the result
        if out is None:
            out = local.new_empty((n_units,) + tail)
        if out.is_contiguous() and tuple(out.shape) == (n_units,) + tail:
            dist.all_gather_into_tensor(out, local, group=group)
            return out
    padded = local.new_zeros((cap,) + tail)
    padded[: local.shape[0]] = local
    buf = local.new_empty((cap * world,) + tail)
    dist.all_gather_into_tensor(buf, padded, group=group)
    parts = []
    for r in range(world):
        a, b = shard_range(n_units, r, world)
        parts.append(buf[r * cap: r * cap + (b - a)])
    res = torch.cat(parts)
    return res if out is None else out.copy_(res)


def compound_angle_shards(iq_local: torch.Tensor, group=None, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Angle sharding (north star (e)): every rank images ITS steering angles
    of the same frames with an ``out="iq"`` plan (the complex sum over its
    transmits, ``das_image(rf[:, a0:a1], plan_over(angles[a0:a1]))`` with
    ``a0, a1 = shard_range(n_angles, rank, world)``); the coherently compounded
    image is the magnitude of the sum over ranks. One all-reduce (SUM) of the
    IQ images — float pairs through ``view_as_real`` — then ``abs``. Equal to
    the one-plan ``out="coherent"`` image up to the order of the FP32 adds.

    ``iq_local`` [F][nz][nx] complex; returns the real image [F][nz][nx] on
    every rank (in ``out`` when given). One rank: just the magnitude."""
    if not iq_local.is_complex():
        raise ValueError("iq_local must be a complex IQ image (plan out='iq')")
    total = iq_local
    if collectives_on(group):
        total = iq_local.clone() if iq_local.is_contiguous() else iq_local.contiguous()
        dist.all_reduce(torch.view_as_real(total), op=dist.ReduceOp.SUM, group=group)
    return torch.abs(total, out=out) if out is not None else torch.abs(total)


def pipelined_gather(compute, n_local: int, out: torch.Tensor, sub: int, group=None,
                     layout: str = "rank_major") -> torch.Tensor:
    """Compute the local units in sub-chunks and all-gather each one as soon as
    it exists, so NVLink moves chunk c while the kernels compute chunk c + 1.

    ``compute(c0, c1)`` returns this rank's units [c0, c1) as a tensor
    [c1 - c0][...] (enqueued on the current stream). Every rank holds the same
    ``n_local`` units; ``out`` [world * n_local][...] receives all of them. Each
    gather is an async NCCL collective ordered after the compute that produced
    its chunk; the call returns once the current stream waits for all of them.

    layout "rank_major": global order (unit f of rank r at ``r * n_local + f``);
    NCCL's list all-gather stages through a flat buffer and copies out.
    layout "chunk_major": chunk [c0, c1) of every rank lands in the contiguous
    slice ``out[world * c0 : world * c1]`` (rank r at ``world * c0 + r * (c1 - c0)``,
    see ``chunk_major_index``) by ``all_gather_into_tensor`` straight into
    ``out`` — no staging buffer, no copy kernel."""
    if layout not in ("rank_major", "chunk_major"):
        raise ValueError(f"layout must be 'rank_major' or 'chunk_major', got {layout!r}")
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if out.shape[0] != world * n_local:
        raise ValueError(f"out holds {out.shape[0]} units, expected world * n_local = {world * n_local}")
    works = []
    for c0 in range(0, n_local, sub):
        c1 = min(n_local, c0 + sub)
        part = compute(c0, c1)
        if not collectives_on(group):
            if part.data_ptr() != out[c0:c1].data_ptr():
                out[c0:c1].copy_(part)
            continue
        if layout == "chunk_major":
            works.append(dist.all_gather_into_tensor(out[world * c0: world * c1], part.contiguous(), group=group,
                                                     async_op=True))
        else:
            views = [out[r * n_local + c0: r * n_local + c1] for r in range(world)]
            works.append(dist.all_gather(views, part.contiguous(), group=group, async_op=True))
    for w in works:
        w.wait()
    return out


def chunk_major_index(f: int, n_local: int, world: int, sub: int) -> int:
    """Position in a ``pipelined_gather(layout="chunk_major")`` output of global
    unit ``f`` (rank ``f // n_local``, local unit ``f % n_local``)."""
    r, i = divmod(int(f), n_local)
    c0 = (i // sub) * sub
    c1 = min(n_local, c0 + sub)
    return world * c0 + r * (c1 - c0) + (i - c0)


def peer_destinations(buffer_ptrs: Sequence[int], rank: int, first_unit: int, unit_bytes: int) -> list:
    """Addresses, in every OTHER rank's copy of a symmetric [n_units][...]
    buffer, of this rank's first unit: where K2's epilogue stores its images."""
    off = int(first_unit) * int(unit_bytes)
    return [int(p) + off for r, p in enumerate(buffer_ptrs) if r != rank]


class PeerImageGather:
    """Image gather fused into K2 (north star (e) over NVLink, no NCCL kernel).

    Every rank holds the whole batch's images in one symmetric-memory buffer
    [n_units][...] (torch symmetric memory: the same allocation mapped into
    every GPU of the node). Rank r images its shard straight into its own slice
    and, from the same epilogue, into the slice of every peer's copy
    (``das_image(..., peers=self.peers)``): the gather traffic leaves the SMs as
    the tiles finish instead of after the last one. ``begin`` / ``end`` are
    device-side barriers over the group on the current stream: nobody
    overwrites a peer's buffer before that peer is done with the previous
    step, and after ``end`` every rank's copy holds every image (the barrier's
    system-scope release / acquire orders the kernel's peer stores)."""

    def __init__(self, n_units: int, unit_shape: Sequence[int], dtype, device, group=None):
        import torch.distributed._symmetric_memory as symm
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        if world - 1 > 7:
            raise ValueError("at most 8 ranks (7 peers per K2 launch)")
        self.buf = symm.empty((n_units, *unit_shape), dtype=dtype, device=device)
        self.handle = symm.rendezvous(self.buf, group if group is not None else dist.group.WORLD)
        self.a, self.b = shard_range(n_units, rank, world)
        unit_bytes = self.buf[0].numel() * self.buf.element_size()
        self.peers = peer_destinations(self.handle.buffer_ptrs, rank, self.a, unit_bytes)

    def local(self) -> torch.Tensor:
        """This rank's slice of its own copy: the ``out`` of its K2 launches."""
        return self.buf[self.a:self.b]

    def begin(self) -> None:
        self.handle.barrier(channel=0)

    def end(self) -> None:
        self.handle.barrier(channel=1)


def try_peer_gather(n_units: int, unit_shape: Sequence[int], dtype, device, group=None):
    """A PeerImageGather if every rank could set one up (agreed over the group,
    so no rank goes on alone), else None — the caller then gathers over NCCL."""
    ok, pg, err = 1, None, None
    try:
        pg = PeerImageGather(n_units, unit_shape, dtype, device, group)
    except Exception as e:  # no symmetric-memory support on this node / build
        ok, err = 0, f"{type(e).__name__}: {e}"
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        t = torch.tensor([ok], device=device, dtype=torch.int32)
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
        ok = int(t.item())
    return (pg if ok else None), err
