"""Oracle geometry: element layout, apertures, delay law, transmit arrival.

Test infrastructure only (see ``oracle/__init__.py``).
"""
from __future__ import annotations

import numpy as np


def element_x(n_el: int, pitch: float) -> np.ndarray:
    """x_n = (n + 0.5) * pitch for n in [-N/2, N/2) — geometry.py:136-150."""
    idx = np.arange(-(n_el // 2), n_el // 2)
    return (idx + 0.5) * pitch


def ref_aperture_half(depth: float, rule: tuple, n_el: int, pitch: float,
                      wavelength: float) -> int:
    """Half count of the array-centred boxcar receive aperture.

    Restates geometry.py:153-199: F# / Kossoff widths convert to the largest even
    count whose extent fits (``2*floor(w/(2p) + 1e-9)``), forced even, clamped to
    [2, N]; FixedCount uses its count directly. The aperture is indices
    [-half, half).  ``rule`` = ("fnumber", f) | ("fixed", n) | ("kossoff", k).
    """
    kind, par = rule
    if kind == "fixed":
        count = int(par)
    else:
        if kind == "fnumber":
            width = depth / par
        elif kind == "kossoff":
            width = np.sqrt(4.0 * wavelength * depth / par)
        else:
            raise TypeError(kind)
        count = 2 * int(np.floor(width / (2.0 * pitch) + 1e-9))
    if count % 2:
        count += 1
    count = max(2, min(count, n_el))
    return count // 2


def receive_delays(x: float, z: float, xs: np.ndarray, c: float) -> np.ndarray:
    """D_n = (z - hypot(x - x_n, z)) / c — das.py:126-132."""
    return (z - np.hypot(x - xs, z)) / c


def focused_tx_arrival(x, z, tx_focus, tx_xs, c):
    """Latest element wavefront of the focused transmit — simulate.py:156-175.

    Vectorised over (x, z) broadcast shapes; tx_xs are the transmit-aperture
    element positions.
    """
    x = np.asarray(x, float)[..., None]
    z = np.asarray(z, float)[..., None]
    focal_delay = (np.hypot(tx_xs, tx_focus) - tx_focus) / c
    travel = np.hypot(x - tx_xs, z) / c
    return np.max(travel - focal_delay, axis=-1)


def focused_expected_arrival(x, z, tx_focus, tx_xs, c):
    """t* = tx arrival + z / c — das.py:135-137."""
    return focused_tx_arrival(x, z, tx_focus, tx_xs, c) + np.asarray(z, float) / c


def plane_wave_expected_arrival(x, z, angle, n_el, pitch, c):
    """t* for a steered plane-wave transmit (NEW, no reference counterpart).

    Convention: the element centres fire in sequence so the
    wavefront is a line at angle ``angle`` to the array; t = 0 is the firing of
    the first element, so the wavefront reaches (x, z) at
    (x sin a + z cos a + (N-1)/2 * pitch * |sin a|) / c.  The receive leg adds
    z / c so that t* - D_n = t_tx + hypot(x - x_n, z) / c, exactly as the
    reference's expected_arrival_time (das.py:135-137) does for focused Tx.
    """
    x = np.asarray(x, float)
    z = np.asarray(z, float)
    s, co = np.sin(angle), np.cos(angle)
    origin = 0.5 * (n_el - 1) * pitch * abs(s)
    return (x * s + z * co + origin) / c + z / c


def hann_weights(x: float, z: float, xs: np.ndarray, f_number: float) -> np.ndarray:
    """Pixel-centred Hann receive apodization of half-width a = z / (2 F#).

    NEW (no reference counterpart; the reference aperture is an array-centred
    boxcar, geometry.py:188-199). w_n = 0.5 (1 + cos(pi (x_n - x) / a)) for
    |x_n - x| < a, else 0.
    """
    a = z / (2.0 * f_number)
    d = xs - x
    w = 0.5 * (1.0 + np.cos(np.pi * d / a))
    return np.where(np.abs(d) < a, w, 0.0)
