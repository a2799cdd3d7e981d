"""tiDAS: reference-native line operator + the north star's row operator.

Reference-native drop-ins (pkg/src/tidas/tidas.py:26-37), float64 on the device:
  tidas_line            tidas.py:493-531  -> K3 (one fixed-profile delayed sum)
                                             + K4 (windowed envelope x theta)
  tidas_psf             tidas.py:317-353  -> K3
  estimate_theta_aligned tidas.py:286-314 -> K3 x 2 + window dots
  theta_row_aligned     tidas.py:464-490  -> GPU synthesis + the above per depth
  TimeWindow, ThetaMatrix, fwhm_window, window_signals (host types / setup)

North-star operators (no reference counterpart, DESIGN.md §tiDAS row operator):
  build_row_kernels      K5: per-depth lateral PSF from the DAS kernel, tiDAS
                         neighbourhood reuse + least-squares theta
  tidas_rowconv          K6: y[b,i,x] = sum_k K[i,k] g[b,i,x+k-H]
  tidas_rowconv_adjoint  K7: g[b,i,x] = sum_k K[i,k] y[b,i,x-k+H]
"""
from __future__ import annotations

import csv
import logging
from dataclasses import dataclass, replace
from pathlib import Path
from typing import Optional, Sequence, Tuple, Union

import numpy as np
import torch

from . import _lib
from . import das as _das
from . import imaging
from .das import Trace, _count, _delayed_sums_dev, _to_dev, _window_read
from .geometry import ApertureRule, DelayProfile, ProbeConfig, rx_aperture, rx_delay_profile
from .metrics import fwhm, window_bounds
from .simulate import RfFrame, ScattererSet, synthesize_frame, tx_arrival_times

__all__ = ["TimeWindow", "ThetaMatrix", "fwhm_window", "window_signals", "estimate_theta_aligned",
           "tidas_psf", "theta_row_aligned", "tidas_line", "build_row_kernels", "lateral_psfs",
           "tidas_rowconv", "tidas_rowconv_adjoint", "rasterize"]

log = logging.getLogger(__name__)


@dataclass(frozen=True)
class TimeWindow:
    """Correction window centre and half-width epsilon [s]."""

    center: float
    half_width: float

    def __post_init__(self) -> None:
        if self.half_width <= 0:
            raise ValueError(f"window half-width must be positive, got {self.half_width}")

    def recenter(self, center: float) -> "TimeWindow":
        return replace(self, center=center)


@dataclass
class ThetaMatrix:
    """theta[reference depth][target depth]; NaN marks failed cells."""

    reference_depths: np.ndarray
    target_depths: np.ndarray
    values: np.ndarray

    def __post_init__(self) -> None:
        self.reference_depths = np.asarray(self.reference_depths, dtype=float)
        self.target_depths = np.asarray(self.target_depths, dtype=float)
        self.values = np.asarray(self.values, dtype=float)
        want = (len(self.reference_depths), len(self.target_depths))
        if self.values.shape != want:
            raise ValueError(f"values shape {self.values.shape} does not match the depth grids {want}")

    def row(self, reference_depth: float) -> np.ndarray:
        return self.values[int(np.argmin(np.abs(self.reference_depths - reference_depth)))]

    def interpolate_row(self, reference_depth: float, depths) -> np.ndarray:
        r = self.row(reference_depth).copy()
        bad = ~np.isfinite(r)
        if bad.any():
            log.warning("theta row at %.4f m: %d missing cells set to 0", reference_depth, bad.sum())
            r[bad] = 0.0
        return np.interp(np.asarray(depths, dtype=float), self.target_depths, r)

    def save_csv(self, path) -> None:
        with open(path, "w", newline="\n") as fh:
            w = csv.writer(fh)
            w.writerow([""] + [f"{d:.9g}" for d in self.target_depths])
            for d, r in zip(self.reference_depths, self.values):
                w.writerow([f"{d:.9g}"] + [f"{v:.9g}" for v in r])

    @classmethod
    def load_csv(cls, path) -> "ThetaMatrix":
        with open(path, newline="") as fh:
            rows = list(csv.reader(fh))
        if len(rows) < 2:
            raise ValueError(f"matrix file {path} has no data rows")
        return cls(np.array([float(r[0]) for r in rows[1:]]),
                   np.array([float(v) for v in rows[0][1:]]),
                   np.array([[float(v) for v in r[1:]] for r in rows[1:]]))


def fwhm_window(focal_psf: Trace, expected_center: float, *,
                min_half_width: Optional[float] = None) -> TimeWindow:
    half = fwhm(focal_psf) / 2.0
    if min_half_width is not None:
        half = max(half, min_half_width)
    if half < 1.0 / focal_psf.sampling_frequency:
        raise ValueError("window half-width is below the sample grid")
    return TimeWindow(center=expected_center, half_width=half)


def window_signals(frame: RfFrame, window: TimeWindow) -> RfFrame:
    t_end = frame.t0 + (frame.n_samples - 1) / frame.sampling_frequency
    if window.center - window.half_width < frame.t0 or window.center + window.half_width > t_end:
        raise ValueError("window lies outside the frame support")
    lo, hi = window_bounds(frame.n_samples, frame.t0, frame.sampling_frequency, window.center,
                           window.half_width)
    if hi <= lo:
        raise ValueError("window covers no sample of the frame")
    masked = np.zeros_like(frame.traces)
    masked[:, lo:hi] = frame.traces[:, lo:hi]
    return RfFrame(masked, frame.sampling_frequency, frame.t0, frame.tx_focus_depth, frame.aperture)


def _profile_sum_dev(frame_d: torch.Tensor, frame: RfFrame, profile: DelayProfile) -> torch.Tensor:
    half = frame.traces.shape[0] // 2
    rows = (np.asarray(profile.element_indices).astype(np.int64) + half)[None, :]
    shifts = (np.asarray(profile.delays, float) * frame.sampling_frequency)[None, :]
    return _delayed_sums_dev(frame_d, rows, shifts)


def estimate_theta_aligned(frame: RfFrame, window: TimeWindow, fixed_delays: DelayProfile,
                           true_delays: DelayProfile, method: str = "linear",
                           _frame_d: Optional[torch.Tensor] = None) -> float:
    """<a, b> / <a, a> of the fixed- and true-profile sums inside the window."""
    if method != "linear":
        a = _das.delayed_sum(frame, fixed_delays.element_indices, fixed_delays.delays, method).samples
        b = _das.delayed_sum(frame, true_delays.element_indices, true_delays.delays, method).samples
        lo, hi = window_bounds(frame.n_samples, frame.t0, frame.sampling_frequency, window.center,
                               window.half_width)
        if hi <= lo:
            raise ValueError("window lies outside the frame support")
        den = float(np.dot(a[lo:hi], a[lo:hi]))
        if den == 0.0:
            raise ZeroDivisionError("window missed the echo: fixed-profile sum has no energy")
        return float(np.dot(a[lo:hi], b[lo:hi])) / den
    L = _lib.lib()
    x_d = _frame_d if _frame_d is not None else _to_dev(np.asarray(frame.traces, float))
    _count(len(fixed_delays) + len(true_delays))
    a = _profile_sum_dev(x_d, frame, fixed_delays)
    b = _profile_sum_dev(x_d, frame, true_delays)
    lo, hi = window_bounds(frame.n_samples, frame.t0, frame.sampling_frequency, window.center,
                           window.half_width)
    if hi <= lo:
        raise ValueError("window lies outside the frame support")
    out = torch.empty(2, dtype=torch.float64, device=x_d.device)
    lo_d = _to_dev(np.array([lo], np.int32), torch.int32)
    hi_d = _to_dev(np.array([hi], np.int32), torch.int32)
    _lib.check(L.tidas_window_dots_f64(_lib.ptr(a), _lib.ptr(b), frame.n_samples, _lib.ptr(lo_d),
                                       _lib.ptr(hi_d), 1, _lib.ptr(out), _lib.stream_handle()))
    ab, aa = out.cpu().numpy()
    if aa == 0.0:
        raise ZeroDivisionError("window missed the echo: fixed-profile sum has no energy")
    return float(ab) / float(aa)


def tidas_psf(windowed_frame: RfFrame, fixed_delays: DelayProfile, theta: float,
              method: str = "linear", crop: bool = False,
              support: Optional[Tuple[int, int]] = None) -> Trace:
    """theta x fixed-profile delayed sum (tidas.py:317-353).

    ``crop`` (linear method) follows the reference's cropped path
    (tidas.py:336-351): the traces are cut to [support0 - span, support1 + 2)
    (span = ceil(-min delay * fs) + 2), each element is shifted with zero fill on
    that segment — so a shift of at least the segment length raises ValueError
    (das.py:87-88) — and the samples outside the segment are 0. ``support``
    ([lo, hi) of the nonzero samples) defaults to the frame's scanned support;
    an all-zero frame gives a zero trace. On the device: the traces are zeroed
    outside the segment and K3 produces only the segment's samples, which is
    bit-identical to the reference's per-segment shifts."""
    if not np.isfinite(theta):
        raise ValueError(f"theta must be finite, got {theta}")
    fs, n, t0 = windowed_frame.sampling_frequency, windowed_frame.n_samples, windowed_frame.t0
    if not (crop and method == "linear"):
        s = _das.delayed_sum(windowed_frame, fixed_delays.element_indices, fixed_delays.delays, method)
        return Trace(theta * s.samples, fs, t0)
    traces = np.asarray(windowed_frame.traces, float)
    if support is None:
        nonzero = np.flatnonzero(np.any(traces != 0.0, axis=0))
        if nonzero.size == 0:
            return Trace(np.zeros(n), fs, t0)
        support = (int(nonzero[0]), int(nonzero[-1]) + 1)
    delays = np.asarray(fixed_delays.delays, float)
    span = int(np.ceil(-delays.min() * fs)) + 2
    lo = max(int(support[0]) - span, 0)
    hi = min(int(support[1]) + 2, n)
    shifts = (delays * fs)[None, :]
    _count(len(delays))
    # the reference shifts a segment of hi - lo samples (das.py:87-88 on that length)
    _das._check_shifts(shifts, max(hi - lo, 0))
    out = torch.zeros((1, n), dtype=torch.float64, device=_das._device())
    if hi > lo:
        x_d = _to_dev(traces)
        x_d[:, :lo] = 0.0
        x_d[:, hi:] = 0.0
        half = traces.shape[0] // 2
        rows = (np.asarray(fixed_delays.element_indices).astype(np.int64) + half)[None, :]
        _delayed_sums_dev(x_d, rows, shifts, np.array([lo]), np.array([hi]), out=out)
    return Trace(theta * out[0].cpu().numpy(), fs, t0)


def theta_row_aligned(reference_depth: float, depth_grid, config: ProbeConfig,
                      tx_rule: ApertureRule, rx_rule: ApertureRule, *, window_half_width: float,
                      tx_focus_depth: Optional[float] = None, spreading: bool = True,
                      method: str = "linear", workers: int = 1) -> np.ndarray:
    """Aligned-window thetas of one reference profile over ``depth_grid``
    (tidas.py:464-490). ``workers`` is accepted; the device runs the cells.

    Every cell's frame is synthesised on the device and stays there (no host
    round trip); the cells' window dot products are collected on the device and
    read back once. Failed cells are NaN with the reference's warning."""
    if method != "linear":  # spectral shifts: the per-cell reference composition
        return _theta_row_per_cell(reference_depth, depth_grid, config, tx_rule, rx_rule,
                                   window_half_width=window_half_width, tx_focus_depth=tx_focus_depth,
                                   spreading=spreading, method=method)
    from .simulate import _synthesize_frame_device
    L = _lib.lib()
    focus = reference_depth if tx_focus_depth is None else tx_focus_depth
    fixed = rx_delay_profile(reference_depth, rx_aperture(reference_depth, rx_rule, config), config)
    fs, c = config.sampling_frequency, config.sound_speed
    depths = np.asarray(depth_grid, dtype=float)
    dots = torch.zeros((len(depths), 2), dtype=torch.float64, device=_das._device())
    failed = {}
    keep = []  # argument tensors stay referenced until their launch is enqueued
    for q, z in enumerate(depths):
        try:
            x_d, aperture = _synthesize_frame_device(ScattererSet.on_axis([z]), focus, config, tx_rule,
                                                     spreading=spreading)
            n = int(x_d.shape[1])
            arrival = float(tx_arrival_times(np.array([z]), focus, aperture, config)[0]) + z / c
            true = rx_delay_profile(z, rx_aperture(z, rx_rule, config), config)
            half = x_d.shape[0] // 2
            prof = []
            for p_ in (fixed, true):
                rows = (np.asarray(p_.element_indices).astype(np.int64) + half)[None, :]
                prof.append(_delayed_sums_dev(x_d, rows, (np.asarray(p_.delays, float) * fs)[None, :]))
            _count(len(fixed) + len(true))
            lo, hi = window_bounds(n, 0.0, fs, arrival, window_half_width)
            if hi <= lo:
                raise ValueError("window lies outside the frame support")
            lo_d = _to_dev(np.array([lo], np.int32), torch.int32)
            hi_d = _to_dev(np.array([hi], np.int32), torch.int32)
            _lib.check(L.tidas_window_dots_f64(_lib.ptr(prof[0]), _lib.ptr(prof[1]), n, _lib.ptr(lo_d),
                                               _lib.ptr(hi_d), 1, _lib.ptr(dots[q]), _lib.stream_handle()))
            keep.append((x_d, prof, lo_d, hi_d))
        except (ValueError, ZeroDivisionError) as exc:
            failed[q] = exc
    ab, aa = dots.cpu().numpy().T  # the one device -> host read of the row
    out = np.full(len(depths), np.nan)
    for q, z in enumerate(depths):
        if q not in failed and aa[q] == 0.0:
            failed[q] = ZeroDivisionError("window missed the echo: fixed-profile sum has no energy")
        if q in failed:
            log.warning("aligned cell (ref %.4f, target %.4f): %s", reference_depth, z, failed[q])
        else:
            out[q] = float(ab[q]) / float(aa[q])
    return out


def _theta_row_per_cell(reference_depth, depth_grid, config, tx_rule, rx_rule, *, window_half_width,
                        tx_focus_depth, spreading, method):
    focus = reference_depth if tx_focus_depth is None else tx_focus_depth
    fixed = rx_delay_profile(reference_depth, rx_aperture(reference_depth, rx_rule, config), config)
    out = []
    for z in np.asarray(depth_grid, dtype=float):
        frame = synthesize_frame(ScattererSet.on_axis([z]), focus, config, tx_rule, spreading=spreading)
        arrival = float(tx_arrival_times(np.array([z]), focus, frame.aperture, config)[0]) + z / config.sound_speed
        true = rx_delay_profile(z, rx_aperture(z, rx_rule, config), config)
        try:
            out.append(estimate_theta_aligned(frame, TimeWindow(arrival, window_half_width), fixed,
                                              true, method))
        except (ValueError, ZeroDivisionError) as exc:
            log.warning("aligned cell (ref %.4f, target %.4f): %s", reference_depth, z, exc)
            out.append(float("nan"))
    return np.array(out)


def tidas_line(frame: RfFrame, fixed_delays: DelayProfile, thetas: Sequence[float], depths,
               config: ProbeConfig, *, window_half_width: float, method: str = "linear") -> np.ndarray:
    """One fixed-profile delayed sum, then per pixel theta x windowed envelope."""
    depths = np.asarray(depths, dtype=float)
    thetas = np.asarray(thetas, dtype=float)
    if len(thetas) != len(depths):
        raise ValueError("one theta per reconstruction depth is required")
    fs, N = frame.sampling_frequency, frame.n_samples
    arrivals = (tx_arrival_times(depths, frame.tx_focus_depth, frame.aperture, config)
                + depths / config.sound_speed)
    lo = np.ceil((arrivals - window_half_width - frame.t0) * fs - 1e-9).astype(np.int64)
    hi = np.floor((arrivals + window_half_width - frame.t0) * fs + 1e-9).astype(np.int64)
    lo, hi = np.maximum(lo, 0), np.minimum(hi, N - 1) + 1
    for k in np.flatnonzero(hi - lo < 4):
        log.warning("pixel at %.4f m: correction window off the trace support", depths[k])
    if method != "linear":
        summed = _das.delayed_sum(frame, fixed_delays.element_indices, fixed_delays.delays, method).samples
        s_d = _to_dev(summed[None])
    else:
        _count(len(fixed_delays))
        s_d = _profile_sum_dev(_to_dev(np.asarray(frame.traces, float)), frame, fixed_delays)
    if len(depths) == 0:
        return np.zeros(0)
    L = _lib.lib()
    P = len(depths)
    out = torch.empty(P, dtype=torch.float64, device=s_d.device)
    tr = torch.zeros(P, dtype=torch.int32, device=s_d.device)
    lo_d = _to_dev(lo.astype(np.int32), torch.int32)
    hi_d = _to_dev(np.maximum(hi, lo).astype(np.int32), torch.int32)
    pos_d = _to_dev((arrivals - frame.t0) * fs)
    th_d = _to_dev(thetas)
    _lib.check(L.tidas_window_envelope_f64(
        _lib.ptr(s_d), N, _lib.ptr(tr), _lib.ptr(lo_d), _lib.ptr(hi_d), _lib.ptr(pos_d),
        _lib.ptr(th_d), P, _lib.ptr(out), _lib.stream_handle()))
    return out.cpu().numpy()


# ------------------------------------------------------------ row operator


def _rowconv(adjoint: bool, x: torch.Tensor, K: torch.Tensor, out=None, stream=None,
             path: str = "auto") -> torch.Tensor:
    L = _lib.lib()
    if x.dtype != torch.float32 or K.dtype != torch.float32:
        raise ValueError("row convolution works on float32 maps and kernels")
    if not (x.is_cuda and K.is_cuda) or x.device != K.device:
        raise ValueError("maps and kernels must be CUDA tensors on one device")
    squeeze = x.dim() == 2
    if squeeze:
        x = x.unsqueeze(0)
    if x.dim() != 3 or K.dim() != 2 or K.shape[0] != x.shape[1]:
        raise ValueError("maps must be [B][nz][nx] and K [nz][taps]")
    x = x.contiguous()
    K = K.contiguous()
    if out is None:
        out = torch.empty_like(x)
    else:
        if squeeze and out.dim() == 2:
            out = out.unsqueeze(0)
        if out.dtype != torch.float32 or out.shape != x.shape or not out.is_contiguous() \
                or out.device != x.device:
            raise ValueError(f"out must be a contiguous float32 tensor of shape {tuple(x.shape)}")
        # the kernels read x rows after writing out rows: in-place is not supported
        xs, xe = x.data_ptr(), x.data_ptr() + x.numel() * 4
        os_, oe = out.data_ptr(), out.data_ptr() + out.numel() * 4
        if xs < oe and os_ < xe:
            raise ValueError("out must not overlap the input maps")
    B, nz, nx = x.shape
    if path not in _lib.ROWCONV_PATHS:
        raise ValueError(f"path must be one of {sorted(_lib.ROWCONV_PATHS)}, got {path!r}")
    _lib.check(L.tidas_rowconv_f32(_lib.ptr(x), _lib.ptr(K), _lib.ptr(out), B, nz, nx, int(K.shape[1]),
                                   int(adjoint), _lib.ROWCONV_PATHS[path], _lib.stream_handle(stream)))
    return out[0] if squeeze else out


def tidas_rowconv(g: torch.Tensor, K: torch.Tensor, out=None, stream=None, path: str = "auto") -> torch.Tensor:
    """K6 forward: y[b,i,x] = sum_k K[i,k] g[b,i,x+k-H] (zero outside).
    ``path``: "auto" (tensor cores when the shape fits), "tensor" or "simt"."""
    return _rowconv(False, g, K, out, stream, path)


def tidas_rowconv_adjoint(y: torch.Tensor, K: torch.Tensor, out=None, stream=None,
                          path: str = "auto") -> torch.Tensor:
    """K7 adjoint: g[b,i,x] = sum_k K[i,k] y[b,i,x-k+H]."""
    return _rowconv(True, y, K, out, stream, path)


def _row_kernels_dev(depths, taps: int, dx: float, *, n_el: int, pitch: float, fs: float, c: float,
                     f0: float, fbw: float, f_number: float, n_samples: int, neighbourhood: int):
    L = _lib.lib()
    dev = torch.device("cuda", torch.cuda.current_device())
    z = torch.as_tensor(np.ascontiguousarray(np.asarray(depths, dtype=np.float64))).to(dev)
    nz = int(z.numel())
    psf = torch.empty((nz, taps), dtype=torch.float64, device=dev)
    K = torch.empty((nz, taps), dtype=torch.float32, device=dev)
    theta = torch.empty(nz, dtype=torch.float64, device=dev)
    _lib.check(L.tidas_build_row_kernels(_lib.ptr(z), nz, int(taps), float(dx), int(n_el), float(pitch), float(fs),
                                         float(c), float(f0), float(fbw), float(f_number), int(n_samples),
                                         int(neighbourhood), _lib.ptr(psf), _lib.ptr(K), _lib.ptr(theta),
                                         _lib.stream_handle()))
    return K, theta, psf


def lateral_psfs(depths, taps: int, dx: float, *, n_el: int, pitch: float, fs: float, c: float,
                 f0: float, fbw: float, f_number: float, n_samples: int) -> torch.Tensor:
    """PSF[i][k] (float64): DAS envelope (0-degree plane wave, Hann F#) at
    (xi_k, z_i) of the RF of a unit scatterer at (0, z_i); xi_k = (k - H) dx.
    K5 (tidas_build_row_kernels): one CTA per depth row, the echo synthesised in
    shared memory and its analytic signal evaluated at the tapped samples by the
    exact discrete Hilbert kernel — no RF frame is materialised."""
    return _row_kernels_dev(depths, taps, dx, n_el=n_el, pitch=pitch, fs=fs, c=c, f0=f0, fbw=fbw,
                            f_number=f_number, n_samples=n_samples, neighbourhood=1)[2]


def build_row_kernels(depths, taps: int, dx: float, *, n_el: int, pitch: float, fs: float,
                      c: float, f0: float, fbw: float, f_number: float, n_samples: int,
                      neighbourhood: int = 8) -> Tuple[torch.Tensor, torch.Tensor]:
    """K5 — per-depth tiDAS row kernels K [nz][taps] (float32) and theta [nz] (float64).

    The lateral PSF of the reference row r(i) (centre of i's block of
    ``neighbourhood`` rows) is reused for every row of the block — the tiDAS
    time-invariance assumption (§tiDAS) applied laterally — and scaled by
    theta_i = <PSF_r, PSF_i> / <PSF_r, PSF_r>, the least-squares weight of
    estimate_theta_aligned (tidas.py:311-314); a zero denominator gives theta 0
    (tidas.py:455-457, experiments.py:399-402). One C-ABI call
    (tidas_build_row_kernels), two kernels, nothing on the host."""
    K, theta, _ = _row_kernels_dev(depths, taps, dx, n_el=n_el, pitch=pitch, fs=fs, c=c, f0=f0, fbw=fbw,
                                   f_number=f_number, n_samples=n_samples, neighbourhood=neighbourhood)
    return K, theta


def rasterize(xs, zs, amps, xgrid, zgrid) -> np.ndarray:
    """Bilinear splat of point reflectivities onto the (z, x) pixel grid (input prep)."""
    xgrid = np.asarray(xgrid, float)
    zgrid = np.asarray(zgrid, float)
    g = np.zeros((len(zgrid), len(xgrid)))
    u = (np.atleast_1d(xs) - xgrid[0]) / (xgrid[1] - xgrid[0])
    v = (np.atleast_1d(zs) - zgrid[0]) / (zgrid[1] - zgrid[0])
    j0 = np.floor(u).astype(np.int64)
    i0 = np.floor(v).astype(np.int64)
    fu, fv = u - j0, v - i0
    a = np.atleast_1d(amps).astype(float)
    for di, wv in ((0, 1.0 - fv), (1, fv)):
        for dj, wu in ((0, 1.0 - fu), (1, fu)):
            ii, jj = i0 + di, j0 + dj
            ok = (ii >= 0) & (ii < len(zgrid)) & (jj >= 0) & (jj < len(xgrid))
            np.add.at(g, (ii[ok], jj[ok]), (a * wv * wu)[ok])
    return g
