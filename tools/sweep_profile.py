"""cProfile of the 600 x 600 error sweep (bench.py's theta_error_sweep line):
host time per function next to the device time.  python tools/sweep_profile.py"""
import cProfile
import pstats
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2507_15464_b200 as tb  # noqa: E402

ROOT = Path(__file__).resolve().parents[1]
d600 = np.linspace(0.005, 0.042, 600)
probe = tb.ProbeConfig()
eps = float(np.load(ROOT / "tests/golden/ref_vectors.npz")["eps"])
run = lambda: tb.error_sweep(d600, probe, tb.Kossoff(0.6), tb.FNumber(1.0), tx_focus_depth=25e-3,  # noqa: E731
                             window_half_width=eps)
run()
torch.cuda.synchronize()
t0 = time.perf_counter()
pr = cProfile.Profile()
pr.enable()
run()
torch.cuda.synchronize()
pr.disable()
print("wall", time.perf_counter() - t0)
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
