"""Time the GPU theta / error sweeps at the paper's scale (600 scatterer depths
x 600 reference profiles; 28.35 min DAS / 21.11 min tiDAS on
the authors' CPU) and at the fixture scale (40 x 40).

  python tools/bench_sweep.py [--n 600] [--reps 2]
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2507_15464_b200 as tb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=600)
ap.add_argument("--reps", type=int, default=2)
args = ap.parse_args()
eps = float(np.load(Path(__file__).resolve().parents[1] / "tests/golden/ref_vectors.npz")["eps"])
probe = tb.ProbeConfig()
res = {}
for n in (40, args.n):
    depths = np.linspace(0.005, 0.042, n)
    for name, fn in (("theta_matrix_sweep", lambda: tb.theta_matrix_sweep(
                         depths, probe, tb.Kossoff(0.6), tb.FNumber(1.0), tx_focus_depth=25e-3,
                         window_half_width=eps)),
                     ("error_sweep", lambda: tb.error_sweep(
                         depths, probe, tb.Kossoff(0.6), tb.FNumber(1.0), tx_focus_depth=25e-3,
                         window_half_width=eps))):
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(args.reps):
            t0 = time.perf_counter()
            out = fn()
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        t = min(ts)
        vals = out.values if hasattr(out, "values") else out[0]
        res[f"{name}_{n}x{n}"] = {"seconds": t, "cells_per_s": n * n / t,
                                  "finite_cells": int(np.isfinite(vals).sum())}
        print(json.dumps({f"{name}_{n}x{n}": res[f"{name}_{n}x{n}"]}), flush=True)
print(json.dumps(res))
