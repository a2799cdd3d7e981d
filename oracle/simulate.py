"""Oracle RF synthesis (seeded inputs for parity tests).

Test infrastructure only (see ``oracle/__init__.py``). Restates the reference
single-scattering model (simulate.py:193-259): every scatterer deposits the
Gaussian-modulated pulse (simulate.py:33-62, sigma from simulate.py:139-153,
support +/- 4 sigma) on every element at tx arrival + return path / c, weighted
by amplitude x z / r (spreading, simulate.py:235/439). The transmit may be the
reference's focused wave or a (NEW) steered plane wave. The trace length is
fixed by the caller (configs pin it) instead of derived from the deepest echo.
"""
from __future__ import annotations

import numpy as np

from . import geom


def pulse_sigma(f0: float, fbw: float) -> float:
    """sqrt(2 ln 2) / (pi * fbw * f0) — simulate.py:139-153."""
    return np.sqrt(2.0 * np.log(2.0)) / (np.pi * fbw * f0)


def pulse_eval(t, f0: float, sigma: float):
    """exp(-t^2 / 2 sigma^2) sin(2 pi f0 t), zero beyond 4 sigma — simulate.py:55-62."""
    t = np.asarray(t, float)
    out = np.exp(-(t * t) / (2.0 * sigma * sigma)) * np.sin(2.0 * np.pi * f0 * t)
    return np.where(np.abs(t) <= 4.0 * sigma, out, 0.0)


def synthesize(sx, sz, amp, *, n_el, pitch, fs, c, f0, fbw, n_samples, tx,
               spreading=True):
    """[n_el][n_samples] float64 RF of point scatterers.

    tx = ("plane", angle_rad) or ("focused", focus_depth, tx_xs).
    """
    sx = np.asarray(sx, float)
    sz = np.asarray(sz, float)
    amp = np.asarray(amp, float)
    xs = geom.element_x(n_el, pitch)
    if tx[0] == "plane":
        arrival = geom.plane_wave_expected_arrival(sx, sz, tx[1], n_el, pitch, c) - sz / c
    elif tx[0] == "focused":
        arrival = geom.focused_tx_arrival(sx, sz, tx[1], tx[2], c)
    else:
        raise ValueError(tx[0])
    dist = np.hypot(sx[:, None] - xs[None, :], sz[:, None])
    tau = arrival[:, None] + dist / c
    w = (sz[:, None] / dist if spreading else np.ones_like(dist)) * amp[:, None]
    sigma = pulse_sigma(f0, fbw)
    half = 4.0 * sigma
    k0 = np.floor((tau - half) * fs).astype(np.int64)
    width = int(np.ceil(2.0 * half * fs)) + 3
    k = k0[..., None] + np.arange(width)
    vals = w[..., None] * pulse_eval(k / fs - tau[..., None], f0, sigma)
    ok = (k >= 0) & (k < n_samples)
    traces = np.zeros((n_el, n_samples))
    rows = np.broadcast_to(np.arange(n_el)[None, :, None], k.shape)
    np.add.at(traces, (rows[ok], k[ok]), vals[ok])
    return traces


def quantize_int16(traces: np.ndarray, target_std: float = 1000.0) -> np.ndarray:
    """Scale to std ``target_std``, round half-even and clip to int16 (cfg5)."""
    std = float(np.std(traces))
    scale = target_std / std if std > 0 else 1.0
    return np.clip(np.rint(traces * scale), -32768, 32767).astype(np.int16)


def speckle(rng: np.random.Generator, n: int, x_range, z_range):
    """n scatterers uniform over the region with N(0,1) amplitudes (cfg2)."""
    sx = rng.uniform(x_range[0], x_range[1], n)
    sz = rng.uniform(z_range[0], z_range[1], n)
    a = rng.standard_normal(n)
    return sx, sz, a
