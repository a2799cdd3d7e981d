"""CPU baseline timing of the reference algorithm — TEST / BENCH INFRASTRUCTURE.

Used only by bench.py's ``cpu_baseline`` leg and ``--impl reference``. Times the
reference's own per-pixel algorithm (das.py:181-193 restated in
oracle/das.py: full-trace two-tap shifts over the aperture, sum, periodic
Hilbert envelope, np.interp) on a bounded, seeded sample of pixels of the
workload, over all host cores like the reference's ``_pmap``
(experiments.py:195-199), and extrapolates to frames/s.
"""
from __future__ import annotations

import os
import time
from concurrent.futures import ProcessPoolExecutor

import numpy as np

from . import das as od
from . import geom

_STATE = {}


def _init(rf, fs, c, pitch, f_number, n_el):
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    _STATE.update(rf=rf, fs=fs, c=c, pitch=pitch, f_number=f_number, n_el=n_el)


def _pixel(args):
    x, z, ts = args
    s = _STATE
    xs_all = geom.element_x(s["n_el"], s["pitch"])
    w_all = geom.hann_weights(x, z, xs_all, s["f_number"])
    keep = np.flatnonzero(w_all > 0.0)
    # full-trace delayed sum over the pixel's aperture (das.py:140-162 restated)
    N = s["rf"].shape[1]
    total = np.zeros(N)
    for e in keep:
        d = (z - np.hypot(x - xs_all[e], z)) / s["c"]
        total += w_all[e] * od.lerp_shift(s["rf"][e], s["fs"], d)
    env = od.envelope(total)
    return od.interp0(ts * s["fs"], env)


def _chunk(items):
    return [_pixel(a) for a in items]


def pixels_per_second(rf, *, fs, c, pitch, f_number, x, z, t_star, n_pixels, seed=0,
                      workers=None, budget_s=None):
    """Time the reference algorithm on ``n_pixels`` seeded pixels of the grid.

    rf: [E][N] one frame (one transmit). Returns (pixels/s, pixels, seconds, workers)."""
    rng = np.random.default_rng(seed)
    iz = rng.integers(0, len(z), n_pixels)
    ix = rng.integers(0, len(x), n_pixels)
    items = [(float(x[j]), float(z[i]), float(t_star[i, j])) for i, j in zip(iz, ix)]
    workers = workers or os.cpu_count() or 1
    n_el = rf.shape[0]
    if workers == 1:
        _init(rf, fs, c, pitch, f_number, n_el)
        t = time.perf_counter()
        _chunk(items)
        dt = time.perf_counter() - t
        return n_pixels / dt, n_pixels, dt, 1
    chunks = [items[k::workers] for k in range(workers)]
    with ProcessPoolExecutor(max_workers=workers, initializer=_init,
                             initargs=(rf, fs, c, pitch, f_number, n_el)) as pool:
        list(pool.map(_chunk, [[items[0]]] * workers))  # warm-up (imports, FFT plans)
        t = time.perf_counter()
        list(pool.map(_chunk, chunks))
        dt = time.perf_counter() - t
    return n_pixels / dt, n_pixels, dt, workers
