"""Oracle DAS: reference full-trace pixel and the exact analytic-signal gather.

Test infrastructure only (see ``oracle/__init__.py``).

Two restatements:

* ``lerp_shift`` / ``delayed_sum`` / ``das_value_fulltrace`` follow the
  reference literally (das.py:82-193): every aperture channel is shifted over the
  whole trace with two-tap linear interpolation and zero fill, summed, the sum's
  periodic Hilbert envelope is taken (metrics.py:30-34 -> scipy.signal.hilbert)
  and sampled with np.interp(left=0, right=0) at t*.  O(channels x samples) per
  pixel, exactly like the reference.
* ``das_image`` is the O(channels) analytic-signal gather:
  one periodic analytic signal per channel, then per pixel two complex beam sums
  C(k0), C(k0+1) of 3 taps per channel and value = (1-f)|C(k0)| + f|C(k0+1)|.
  It equals ``das_value_fulltrace`` to rounding whenever each channel holds at
  least max|shift|+1 leading zeros (zero-fill shift == circular shift).
"""
from __future__ import annotations

import numpy as np
import scipy.fft as sp_fft

from . import geom

# ---------------------------------------------------------------- analytic


def hilbert_multiplier(n: int) -> np.ndarray:
    """h of scipy.signal.hilbert: [1, 2..2, 1 (Nyquist, even n), 0..]."""
    h = np.zeros(n)
    if n % 2 == 0:
        h[0] = h[n // 2] = 1.0
        h[1:n // 2] = 2.0
    else:
        h[0] = 1.0
        h[1:(n + 1) // 2] = 2.0
    return h


def analytic_signal(x: np.ndarray) -> np.ndarray:
    """Periodic analytic signal along the last axis (metrics.py:30-34 semantics).

    Uses scipy.fft, the transform scipy.signal.hilbert itself calls
    (scipy/signal/_signaltools.py, scipy 1.18.1 here; the reference pins only
    scipy>=1.10, pkg/pyproject.toml:12), so the oracle's envelopes match the
    reference's to the last few ulps.
    """
    x = np.asarray(x, dtype=float)
    n = x.shape[-1]
    return sp_fft.ifft(sp_fft.fft(x, axis=-1) * hilbert_multiplier(n), axis=-1)


def envelope(x: np.ndarray) -> np.ndarray:
    """|analytic| — metrics.py:30-34 (ValueError below 4 samples)."""
    if np.shape(x)[-1] < 4:
        raise ValueError("envelope needs at least 4 samples")
    return np.abs(analytic_signal(x))


# ----------------------------------------------------- reference full trace


def split_shift(shift: float):
    """(m, mu, integer?) for a sample shift — das.py:89-97 (integer rule 1e-9)."""
    nearest = round(shift)
    if abs(shift - nearest) < 1e-9:
        return int(nearest), 0.0, True
    m = int(np.floor(shift))
    return m, shift - m, False


def lerp_shift(x: np.ndarray, fs: float, delay: float) -> np.ndarray:
    """out[k] = (1-mu) x~[k-m] + mu x~[k-m-1] with zero fill — das.py:82-107."""
    n = len(x)
    if abs(delay) * fs >= n:
        raise ValueError("delay exceeds the trace support")
    m, mu, integer = split_shift(delay * fs)
    out = np.zeros(n)
    if integer:
        if m >= 0:
            out[m:] = x[:n - m]
        else:
            out[:n + m] = x[-m:]
        return out
    k = np.arange(n)
    a = k - m
    b = k - m - 1
    xa = np.where((a >= 0) & (a < n), x[np.clip(a, 0, n - 1)], 0.0)
    xb = np.where((b >= 0) & (b < n), x[np.clip(b, 0, n - 1)], 0.0)
    return (1.0 - mu) * xa + mu * xb


def delayed_sum(traces: np.ndarray, fs: float, element_indices, delays) -> np.ndarray:
    """Sequential sum over the aperture of lerp-shifted rows — das.py:140-149."""
    half = traces.shape[0] // 2
    total = np.zeros(traces.shape[1])
    for idx, d in zip(element_indices, delays):
        total += lerp_shift(traces[int(idx) + half], fs, d)
    return total


def interp0(pos: float, values: np.ndarray) -> float:
    """np.interp(pos, arange(n), values, left=0, right=0) — das.py:173."""
    return float(np.interp(pos, np.arange(len(values)), values, left=0.0, right=0.0))


def das_value_fulltrace(traces, fs, t0, x, z, ap_half, pitch, c, t_star,
                        weights=None):
    """Reference das_value (das.py:181-193) for an array-centred boxcar aperture
    [-ap_half, ap_half) (optionally weighted, for the Hann restatement)."""
    n_el = traces.shape[0]
    idx = np.arange(-ap_half, ap_half)
    xs = (idx + 0.5) * pitch
    delays = geom.receive_delays(x, z, xs, c)
    half = n_el // 2
    total = np.zeros(traces.shape[1])
    for j, (n, d) in enumerate(zip(idx, delays)):
        w = 1.0 if weights is None else weights[j]
        if w == 0.0:
            continue
        total += w * lerp_shift(traces[n + half], fs, d)
    env = envelope(total)
    return interp0((t_star - t0) * fs, env)


# ------------------------------------------------------ analytic gather (B.1)


def _gather_iq(A, fs, t0, x, z, t_star, idx, weights, pitch, c):
    """(C0, C1, k0, f) of one pixel; A is [n_el][N] complex analytic RF."""
    n_el, n = A.shape
    pos = (t_star - t0) * fs
    if pos < 0.0 or pos > n - 1:
        return 0.0, 0.0, 0, 0.0, False
    k0 = int(np.floor(pos))
    f = pos - k0
    xs = (idx + 0.5) * pitch
    delays = geom.receive_delays(x, z, xs, c)
    c0 = 0.0 + 0.0j
    c1 = 0.0 + 0.0j
    half = n_el // 2
    for n_i, d, w in zip(idx, delays, weights):
        if w == 0.0:
            continue
        m, mu, _ = split_shift(d * fs)
        row = A[n_i + half]
        a_m1 = row[(k0 - m - 1) % n]
        a_0 = row[(k0 - m) % n]
        a_p1 = row[(k0 - m + 1) % n]
        c0 += w * ((1.0 - mu) * a_0 + mu * a_m1)
        c1 += w * ((1.0 - mu) * a_p1 + mu * a_0)
    return c0, c1, k0, f, True


def das_image(A, fs, t0, xgrid, zgrid, pitch, c, t_star, aperture, out="envelope"):
    """Analytic-gather DAS image, float64.

    A        : [n_angles][n_el][N] complex analytic RF (one frame)
    t_star   : [n_angles][nz][nx] expected arrival per pixel and transmit
    aperture : ("ref", rule, wavelength) array-centred boxcar (reference) or
               ("hann", f_number) pixel-centred Hann F# (north star)
    out      : "envelope" — per angle (1-f)|C0| + f|C1| (reference two-stage
               interpolation), summed over angles (incoherent for >1 angle);
               "iq" — complex (1-f) C0 + f C1 summed over angles;
               "coherent" — |iq|.
    returns  : [nz][nx] float64 (complex for "iq").
    """
    A = np.asarray(A)
    n_ang, n_el, _ = A.shape
    xs_all = geom.element_x(n_el, pitch)
    nz, nx = len(zgrid), len(xgrid)
    res = np.zeros((nz, nx), dtype=complex if out == "iq" else float)
    idx_all = np.arange(-(n_el // 2), n_el // 2)
    for iz, z in enumerate(zgrid):
        if aperture[0] == "ref":
            half = geom.ref_aperture_half(z, aperture[1], n_el, pitch, aperture[2])
            idx = np.arange(-half, half)
        for ix, x in enumerate(xgrid):
            if aperture[0] == "hann":
                w_all = geom.hann_weights(x, z, xs_all, aperture[1])
                keep = w_all > 0.0
                idx, w = idx_all[keep], w_all[keep]
            else:
                w = np.ones(len(idx))
            acc_iq = 0.0 + 0.0j
            acc_env = 0.0
            for a in range(n_ang):
                c0, c1, _, f, ok = _gather_iq(A[a], fs, t0, x, z, t_star[a, iz, ix],
                                              idx, w, pitch, c)
                if not ok:
                    continue
                acc_env += (1.0 - f) * abs(c0) + f * abs(c1)
                acc_iq += (1.0 - f) * c0 + f * c1
            if out == "envelope":
                res[iz, ix] = acc_env
            elif out == "iq":
                res[iz, ix] = acc_iq
            elif out == "coherent":
                res[iz, ix] = abs(acc_iq)
            else:
                raise ValueError(out)
    return res


def das_image_vectorized(A, fs, t0, xgrid, zgrid, pitch, c, t_star, f_number,
                         out="envelope"):
    """Same as ``das_image`` for the Hann aperture, vectorised over pixels.

    Used at the larger parity sizes (cfg1/cfg2 grids) where the per-pixel loop
    would be slow; checked against ``das_image`` in tests.
    """
    A = np.asarray(A)
    n_ang, n_el, n = A.shape
    xs = geom.element_x(n_el, pitch)
    Z, X = np.meshgrid(np.asarray(zgrid, float), np.asarray(xgrid, float), indexing="ij")
    acc_env = np.zeros(Z.shape)
    acc_iq = np.zeros(Z.shape, complex)
    for a in range(n_ang):
        pos = (t_star[a] - t0) * fs
        valid = (pos >= 0.0) & (pos <= n - 1)
        k0 = np.floor(np.where(valid, pos, 0.0)).astype(np.int64)
        f = np.where(valid, pos - k0, 0.0)
        c0 = np.zeros(Z.shape, complex)
        c1 = np.zeros(Z.shape, complex)
        for e in range(n_el):
            d = xs[e] - X
            ap = Z / (2.0 * f_number)
            inside = np.abs(d) < ap
            if not inside.any():
                continue
            w = np.where(inside, 0.5 * (1.0 + np.cos(np.pi * d / ap)), 0.0)
            shift = (Z - np.hypot(X - xs[e], Z)) / c * fs
            nearest = np.round(shift)
            integer = np.abs(shift - nearest) < 1e-9
            m = np.where(integer, nearest, np.floor(shift)).astype(np.int64)
            mu = np.where(integer, 0.0, shift - np.floor(shift))
            row = A[a, e]
            am1 = row[(k0 - m - 1) % n]
            a0 = row[(k0 - m) % n]
            ap1 = row[(k0 - m + 1) % n]
            c0 += w * ((1.0 - mu) * a0 + mu * am1)
            c1 += w * ((1.0 - mu) * ap1 + mu * a0)
        c0 = np.where(valid, c0, 0.0)
        c1 = np.where(valid, c1, 0.0)
        acc_env += (1.0 - f) * np.abs(c0) + f * np.abs(c1)
        acc_iq += (1.0 - f) * c0 + f * c1
    if out == "envelope":
        return acc_env
    if out == "iq":
        return acc_iq
    if out == "coherent":
        return np.abs(acc_iq)
    raise ValueError(out)


def rel_l2(a, b) -> float:
    a = np.asarray(a)
    b = np.asarray(b)
    den = np.sqrt(np.sum(np.abs(b) ** 2))
    return float(np.sqrt(np.sum(np.abs(a - b) ** 2)) / den) if den > 0 else float(
        np.sqrt(np.sum(np.abs(a) ** 2)))


def global_error(reference, candidate) -> float:
    """||cand - ref||^2 / ||ref||^2 — metrics.py:105-112."""
    reference = np.asarray(reference, float)
    candidate = np.asarray(candidate, float)
    den = float(np.sum(reference ** 2))
    if den == 0.0:
        raise ValueError("reference carries no energy")
    return float(np.sum((candidate - reference) ** 2)) / den
