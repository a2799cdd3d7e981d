"""K1 (rf_analytic) timing at the three register four-step lengths, optionally
with a variant library (tools/build_variant.sh):

  python tools/k1_time.py [lib.so]

cfg2: 256 frames x 128 ch x 4096 f32; cfg5: 64 frames x 192 ch x 8192 int16;
cfg1: 256 frames x 64 ch x 2048 f64. Prints microseconds per frame and a
checksum (bitwise comparisons between variants: the checksum of |A|)."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2507_15464_b200 import _lib  # noqa: E402

if len(sys.argv) > 1:
    _lib.load(Path(sys.argv[1]))
import paper_2507_15464_b200 as tb  # noqa: E402


def t(fn, frames, n=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / n / frames


g = torch.Generator(device="cuda").manual_seed(7)
res = {"lib": sys.argv[1] if len(sys.argv) > 1 else "default"}
for name, F, E, N, dt in (("cfg2", 256, 128, 4096, torch.float32), ("cfg5", 64, 192, 8192, torch.int16),
                          ("cfg1", 256, 64, 2048, torch.float64)):
    x = torch.randn((F, 1, E, N), device="cuda", generator=g) * (1000.0 if dt == torch.int16 else 1.0)
    x = x.round().to(dt) if dt == torch.int16 else x.to(dt)
    an = torch.empty((F, 1, E, N), dtype=torch.complex64, device="cuda")
    us = t(lambda: tb.rf_analytic(x, "f32", out=an), F)
    res[name] = {"us_per_frame": round(us, 4), "checksum": float(an.abs().double().sum())}
    del x, an
print(json.dumps(res), flush=True)
