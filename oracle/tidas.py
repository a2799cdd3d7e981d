"""Oracle tiDAS: reference-native line reconstruction, theta, row operators.

Test infrastructure only (see ``oracle/__init__.py``).

Reference-native (pinned by the reference):
  window_bounds        metrics.py:78-82
  tidas_line           tidas.py:493-531
  estimate_theta_aligned tidas.py:286-314
  theta_row_aligned    tidas.py:432-490 (serial)
  reference_frame      simulate.py:193-259 (focused transmit, derived length)

North-star-only (unpinned; DESIGN.md §tiDAS row operator):
  rowconv_fwd / rowconv_adj   y[b,i,x] = sum_k K[i,k] g[b,i,x+k-H]
  build_row_kernels           per-depth lateral PSF of a unit scatterer, tiDAS
                              neighbourhood reuse + least-squares theta
"""
from __future__ import annotations

import numpy as np

from . import das as odas
from . import geom
from . import simulate as osim


def window_bounds(n: int, t0: float, fs: float, center: float, half_width: float):
    """Half-open [lo, hi) of samples inside center +/- half_width — metrics.py:78-82."""
    lo = int(np.ceil((center - half_width - t0) * fs - 1e-9))
    hi = int(np.floor((center + half_width - t0) * fs + 1e-9))
    return max(lo, 0), min(hi, n - 1) + 1


def windowed_envelope_value(summed, fs, t0, t_star, half_width):
    """Envelope of summed[lo:hi] sampled at t* (das.py:174-178; tidas.py:523-530)."""
    n = len(summed)
    lo, hi = window_bounds(n, t0, fs, t_star, half_width)
    if hi - lo < 4:
        return 0.0
    env = odas.envelope(summed[lo:hi])
    return odas.interp0((t_star - t0) * fs - lo, env)


def tidas_line(traces, fs, t0, fixed_idx, fixed_delays, thetas, t_stars, half_width):
    """tidas.py:493-531 with precomputed on-axis arrivals t_stars."""
    summed = odas.delayed_sum(traces, fs, fixed_idx, fixed_delays)
    return np.array([th * windowed_envelope_value(summed, fs, t0, ts, half_width)
                     for th, ts in zip(thetas, t_stars)])


def estimate_theta_aligned(traces, fs, t0, center, half_width, fixed_idx, fixed_delays,
                           true_idx, true_delays):
    """<a, b> / <a, a> over window_bounds — tidas.py:286-314."""
    a = odas.delayed_sum(traces, fs, fixed_idx, fixed_delays)
    b = odas.delayed_sum(traces, fs, true_idx, true_delays)
    lo, hi = window_bounds(traces.shape[1], t0, fs, center, half_width)
    if hi <= lo:
        raise ValueError("window lies outside the frame support")
    den = float(np.dot(a[lo:hi], a[lo:hi]))
    if den == 0.0:
        raise ZeroDivisionError("window missed the echo")
    return float(np.dot(a[lo:hi], b[lo:hi])) / den


def reference_frame(depth, tx_focus, *, n_el, pitch, fs, c, f0, fbw, tx_half):
    """Unit on-axis scatterer frame with the reference's derived length.

    simulate.py:193-259: n_samples = ceil((tau_max + 8 sigma) fs) + 1.
    """
    xs = geom.element_x(n_el, pitch)
    tx_xs = (np.arange(-tx_half, tx_half) + 0.5) * pitch
    arrival = geom.focused_tx_arrival(0.0, depth, tx_focus, tx_xs, c)
    tau = arrival + np.hypot(0.0 - xs, depth) / c
    sigma = osim.pulse_sigma(f0, fbw)
    n = int(np.ceil((tau.max() + 8.0 * sigma) * fs)) + 1
    return osim.synthesize([0.0], [depth], [1.0], n_el=n_el, pitch=pitch, fs=fs, c=c,
                           f0=f0, fbw=fbw, n_samples=n,
                           tx=("focused", tx_focus, tx_xs)), tx_xs


def theta_row_aligned(ref_depth, depths, *, n_el, pitch, fs, c, f0, fbw, tx_rule,
                      rx_rule, half_width, tx_focus=None):
    """tidas.py:464-490 (serial). Failed cells -> NaN."""
    focus = ref_depth if tx_focus is None else tx_focus
    wl = c / f0
    tx_half = geom.ref_aperture_half(focus, tx_rule, n_el, pitch, wl)
    fh = geom.ref_aperture_half(ref_depth, rx_rule, n_el, pitch, wl)
    f_idx = np.arange(-fh, fh)
    f_del = geom.receive_delays(0.0, ref_depth, (f_idx + 0.5) * pitch, c)
    out = []
    for z in np.asarray(depths, float):
        traces, tx_xs = reference_frame(z, focus, n_el=n_el, pitch=pitch, fs=fs, c=c,
                                        f0=f0, fbw=fbw, tx_half=tx_half)
        center = float(geom.focused_expected_arrival(0.0, z, focus, tx_xs, c))
        th = geom.ref_aperture_half(z, rx_rule, n_el, pitch, wl)
        t_idx = np.arange(-th, th)
        t_del = geom.receive_delays(0.0, z, (t_idx + 0.5) * pitch, c)
        try:
            out.append(estimate_theta_aligned(traces, fs, 0.0, center, half_width,
                                              f_idx, f_del, t_idx, t_del))
        except (ValueError, ZeroDivisionError):
            out.append(float("nan"))
    return np.array(out)


# ------------------------------------------------------- row operators (new)


def rowconv_fwd(g: np.ndarray, K: np.ndarray) -> np.ndarray:
    """y[..., i, x] = sum_k K[i, k] g[..., i, x + k - H], zero outside, float64."""
    g = np.asarray(g, float)
    K = np.asarray(K, float)
    T = K.shape[1]
    H = (T - 1) // 2
    nx = g.shape[-1]
    pad = np.zeros(g.shape[:-1] + (nx + 2 * H,))
    pad[..., H:H + nx] = g
    y = np.zeros_like(g)
    for k in range(T):
        y += K[:, k][:, None] * pad[..., k:k + nx]
    return y


def rowconv_adj(y: np.ndarray, K: np.ndarray) -> np.ndarray:
    """g[..., i, x] = sum_k K[i, k] y[..., i, x - k + H] (exact adjoint of fwd)."""
    y = np.asarray(y, float)
    K = np.asarray(K, float)
    T = K.shape[1]
    H = (T - 1) // 2
    nx = y.shape[-1]
    pad = np.zeros(y.shape[:-1] + (nx + 2 * H,))
    pad[..., H:H + nx] = y
    g = np.zeros_like(y)
    for k in range(T):
        # x - k + H  ->  padded index x - k + 2H
        g += K[:, k][:, None] * pad[..., 2 * H - k:2 * H - k + nx]
    return g


def neighbourhood_reference_rows(n_rows: int, nb: int) -> np.ndarray:
    """Row whose PSF shape serves row i: centre of its block of ``nb`` rows."""
    i = np.arange(n_rows)
    r = (i // nb) * nb + nb // 2
    return np.minimum(r, n_rows - 1)


def lateral_psfs(depths, taps, dx, *, n_el, pitch, fs, c, f0, fbw, f_number, n_samples):
    """PSF[i][k]: DAS envelope at (xi_k, z_i) of a unit scatterer at (0, z_i).

    0-degree plane-wave transmit, pixel-centred Hann F# receive, analytic gather
    (das.das_image_vectorized) — the same DAS the image path computes.
    """
    H = (taps - 1) // 2
    xi = (np.arange(taps) - H) * dx
    out = np.zeros((len(depths), taps))
    for i, z in enumerate(np.asarray(depths, float)):
        rf = osim.synthesize([0.0], [z], [1.0], n_el=n_el, pitch=pitch, fs=fs, c=c,
                             f0=f0, fbw=fbw, n_samples=n_samples, tx=("plane", 0.0))
        A = odas.analytic_signal(rf)[None]
        ts = geom.plane_wave_expected_arrival(xi[None, :], np.array([[z]]), 0.0, n_el,
                                              pitch, c)[None]
        out[i] = odas.das_image_vectorized(A, fs, 0.0, xi, [z], pitch, c, ts,
                                           f_number)[0]
    return out


def build_row_kernels_from_psfs(psf: np.ndarray, nb: int):
    """K[i] = theta_i * PSF[r(i)], theta_i = <PSF_r, PSF_i> / <PSF_r, PSF_r>.

    Least-squares form of estimate_theta_aligned (tidas.py:311-314); a zero
    denominator becomes NaN -> 0 as the reference's row consumers do
    (tidas.py:455-457, experiments.py:399-402).
    """
    psf = np.asarray(psf, float)
    r = neighbourhood_reference_rows(psf.shape[0], nb)
    a = psf[r]
    den = np.sum(a * a, axis=1)
    num = np.sum(a * psf, axis=1)
    with np.errstate(invalid="ignore", divide="ignore"):
        theta = np.where(den > 0.0, num / np.where(den > 0.0, den, 1.0), 0.0)
    return theta[:, None] * a, theta


def rasterize(sx, sz, amp, xgrid, zgrid) -> np.ndarray:
    """Bilinear splat of point reflectivities onto the (z, x) pixel grid."""
    xgrid = np.asarray(xgrid, float)
    zgrid = np.asarray(zgrid, float)
    g = np.zeros((len(zgrid), len(xgrid)))
    dxg = xgrid[1] - xgrid[0]
    dzg = zgrid[1] - zgrid[0]
    for x, z, a in zip(np.atleast_1d(sx), np.atleast_1d(sz), np.atleast_1d(amp)):
        u = (x - xgrid[0]) / dxg
        v = (z - zgrid[0]) / dzg
        j0, i0 = int(np.floor(u)), int(np.floor(v))
        fu, fv = u - j0, v - i0
        for di, wv in ((0, 1.0 - fv), (1, fv)):
            for dj, wu in ((0, 1.0 - fu), (1, fu)):
                i, j = i0 + di, j0 + dj
                if 0 <= i < len(zgrid) and 0 <= j < len(xgrid):
                    g[i, j] += a * wv * wu
    return g
