import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_2507_15464_b200 as T
from paper_2507_15464_b200 import tidas as tt
p1 = T.ProbeConfig(element_count=64, pitch=0.3e-3, center_frequency=5e6, sampling_frequency=20e6, sound_speed=1540.0, fractional_bandwidth=0.6)
g = np.load('tests/golden/ref_vectors.npz')
d1 = np.linspace(5e-3, 40e-3, 256)
for k in range(3):
    t0 = time.perf_counter()
    th = T.theta_row_aligned(20e-3, d1, p1, T.FixedCount(64), T.FNumber(1.5), window_half_width=float(g["C1_eps"]))
    t1 = time.perf_counter()
    th2 = tt._theta_row_per_cell(20e-3, d1, p1, T.FixedCount(64), T.FNumber(1.5), window_half_width=float(g["C1_eps"]), tx_focus_depth=None, spreading=True, method="linear")
    t2 = time.perf_counter()
    print("batched %.3f s  per-cell %.3f s  equal %s" % (t1 - t0, t2 - t1, np.array_equal(np.nan_to_num(th, nan=-1), np.nan_to_num(th2, nan=-1))))
ref = np.where(np.isfinite(th), th, 0.0)
print("vs golden C1_theta", np.max(np.abs(ref - g["C1_theta"])))
