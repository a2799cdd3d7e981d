"""Subprocess of tests/test_gpu_peers.py: a 1-rank NCCL group, a symmetric
image buffer (parallel.PeerImageGather) and K2 writing into it through the
symmetric mapping's address. Prints one JSON line."""
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    from tests.setups import CFG2, grid
    import paper_2507_15464_b200 as tb
    from paper_2507_15464_b200 import parallel
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(parallel.free_port()), RANK="0", WORLD_SIZE="1",
                      LOCAL_RANK="0")
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    cfg = CFG2
    F, nz, nx = 9, 33, 47
    x, z = grid(cfg, nz, nx)
    plan = tb.plane_wave_plan(n_el=cfg["n_el"], pitch=cfg["pitch"], fs=cfg["fs"], c=cfg["c"],
                              n_samples=cfg["n_samples"], x=x, z=z)
    g = torch.Generator(device="cuda").manual_seed(5)
    rf = torch.randn((F, 1, cfg["n_el"], cfg["n_samples"]), device="cuda", generator=g)
    ref = tb.das_image(rf, plan)
    pg, err = parallel.try_peer_gather(F, (nz, nx), torch.float32, torch.device("cuda", 0))
    if pg is None:
        print(json.dumps({"skip": err}), flush=True)
        return 0
    assert pg.peers == [] and (pg.a, pg.b) == (0, F)
    pg.buf.zero_()
    # the own mapping's address as the peer destination, a plain tensor as out
    own = [int(pg.handle.buffer_ptrs[0])]
    out = torch.empty_like(ref)
    pg.begin()
    tb.das_image(rf, plan, out=out, peers=own)
    pg.end()
    torch.cuda.synchronize()
    ok = bool(torch.equal(out, ref)) and bool(torch.equal(pg.buf, ref))
    # and the bench's form: images straight into local(), no peers at world 1
    pg.buf.zero_()
    pg.begin()
    tb.das_image(rf, plan, out=pg.local(), peers=pg.peers)
    pg.end()
    torch.cuda.synchronize()
    ok = ok and bool(torch.equal(pg.buf, ref))
    print(json.dumps({"ok": ok}), flush=True)
    dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
