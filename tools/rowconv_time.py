"""Row operator timings (tcgen05 path): cfg4 forward / adjoint (256 maps of
2048 x 1024) and cfg2 maps (512 x 512 x 256), CUDA events, HBM fraction."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2507_15464_b200 as tb  # noqa: E402
from paper_2507_15464_b200 import _lib  # noqa: E402

if len(sys.argv) > 1:  # a variant library (tools/build_variant.sh)
    _lib.load(Path(sys.argv[1]))

HBM = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] \
    if (Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").exists() else 6650.0


def t(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


g = torch.Generator(device="cuda").manual_seed(3)
for name, (B, nz, nx) in {"cfg4": (256, 2048, 1024), "cfg2": (512, 512, 256)}.items():
    x = (torch.rand((B, nz, nx), device="cuda", generator=g) < 0.02).float() * torch.randn((B, nz, nx), device="cuda", generator=g)
    K = torch.randn((nz, 129), device="cuda", generator=g) / 16
    y, a = torch.empty_like(x), torch.empty_like(x)
    tb.tidas_rowconv(x, K, out=y, path="tensor")
    tf = t(lambda: tb.tidas_rowconv(x, K, out=y, path="tensor"))
    ta = t(lambda: tb.tidas_rowconv_adjoint(y, K, out=a, path="tensor"))
    tfd = t(lambda: tb.tidas_rowconv(y, K, out=a, path="tensor"))  # forward on dense input (y)
    byt = B * nz * nx * 8 + K.numel() * 4
    print(json.dumps({"lib": sys.argv[1] if len(sys.argv) > 1 else "default", name: {"fwd_ms": tf, "adj_ms": ta, "fwd_frac": byt / tf / 1e6 / HBM,
                             "adj_frac": byt / ta / 1e6 / HBM, "fwd_dense_ms": tfd, "maps_per_s_fwd": B / tf * 1e3,
                             "checksum_fwd": float(a.double().abs().sum())}}), flush=True)
    del x, y, a
