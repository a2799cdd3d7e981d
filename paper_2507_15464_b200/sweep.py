"""FFT theta estimator and the theta / error sweeps on the GPU.

Drop-ins for the reference's
  estimate_theta      tidas.py:237-283 (with _windowed_spectra / _delay_phases)
  theta_matrix_sweep  tidas.py:394-425 (one single-scatterer frame per column)
and ``error_sweep``, the (theta, local error, global error) matrices that
``run_error_sweep`` (experiments.py:299-361) writes as theta_matrix.csv,
error_local.csv, error_global.csv and error_mask.csv.

All columns of a sweep are simulated in one launch (tidas_synthesize, FP64),
windowed and support-scanned in one launch, their window spectra computed once
per (column, FFT length) and cached in HBM, and every cell's theta computed by
one CTA (tidas_theta_cells_f64). The error sweep adds the true-profile PSF per
column and the cropped fixed-profile PSF per cell (K3, bit-identical to numpy)
and one reduction per cell (tidas_psf_errors_f64). Host work is the geometry
(apertures, delay profiles, FFT lengths) in float64 — O(cells x aperture).
Failure cases become NaN cells exactly as in the reference.
"""
from __future__ import annotations

from typing import Optional, Tuple

import numpy as np
import torch

from . import _lib
from . import das as _das
from .geometry import (ApertureRule, DelayProfile, ProbeConfig, aperture_half_counts, element_positions,
                       tx_aperture)
from .metrics import window_bounds
from .simulate import RfFrame, _focused_arrivals, _synth_device, make_pulse

FORMS = {"beamsum": 0, "per_element": 1}
_COL_BATCH = 96  # columns per device batch (bounds the spectra / PSF scratch)


def _next_pow2(n: int) -> int:
    return 1 << max(int(n) - 1, 0).bit_length()


def _dev():
    _lib.lib()
    return torch.device("cuda", torch.cuda.current_device())


def _i32(a, dev):
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.int32)).to(dev)


def _f64(a, dev):
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64)).to(dev)


class _Columns:
    """Single on-axis scatterer frames (one per target depth), windowed on the device."""

    def __init__(self, targets, config: ProbeConfig, tx_rule: ApertureRule, tx_focus: float,
                 half_width: float, spreading: bool):
        dev = _dev()
        self.targets = np.asarray(targets, float)
        T = len(self.targets)
        c, fs, n_el = config.sound_speed, config.sampling_frequency, config.element_count
        self.fs, self.n_el = fs, n_el
        pulse = make_pulse(config)
        ap = tx_aperture(tx_focus, tx_rule, config)
        arr = _focused_arrivals(np.zeros(T), self.targets, tx_focus, ap, config)  # [T]
        xs = element_positions(np.arange(-n_el // 2, n_el // 2), config)
        dist = np.hypot(xs[None, :], self.targets[:, None])
        # frame length of synthesize_frame (simulate.py:229)
        self.n_len = (np.ceil(((arr[:, None] + dist / c).max(axis=1) + pulse.duration) * fs)).astype(np.int64) + 1
        self.N = int(self.n_len.max())
        frames = _synth_device(np.zeros((T, 1)), self.targets[:, None], np.ones((T, 1)), arr[:, None, None],
                               n_frames=T, n_angles=1, n_el=n_el, pitch=config.pitch, c=c, fs=fs,
                               f0=pulse.center_frequency, fbw=pulse.fractional_bandwidth,
                               n_samples=self.N, spreading=spreading, dtype=torch.float64, device=dev)
        # one extra all-zero row at the end: padding target for K3 profiles
        flat = torch.zeros((T * n_el + 1, self.N), dtype=torch.float64, device=dev)
        flat[: T * n_el] = frames.reshape(T * n_el, self.N)
        del frames
        self.flat = flat
        self.zero_row = T * n_el
        # window per column (tidas.py:150-168 / experiments.py:305-313): centred on
        # the focused-transmit arrival + z / c (das.expected_arrival_time, and
        # tx_arrival_times(...)[0] + z / c in tidas.py:369-371 — the same value)
        centers = arr + self.targets / c
        self.centers = centers
        self.ok = np.ones(T, bool)
        self.wlo = np.zeros(T, np.int32)
        self.whi = np.zeros(T, np.int32)
        for t in range(T):
            n = int(self.n_len[t])
            t_end = (n - 1) / fs
            lo, hi = window_bounds(n, 0.0, fs, float(centers[t]), half_width)
            if centers[t] - half_width < 0.0 or centers[t] + half_width > t_end or hi <= lo:
                self.ok[t] = False
                lo = hi = 0
            self.wlo[t], self.whi[t] = lo, hi
        first = torch.empty((T, n_el), dtype=torch.int32, device=dev)
        last = torch.empty((T, n_el), dtype=torch.int32, device=dev)
        lo_d, hi_d = _i32(self.wlo, dev), _i32(self.whi, dev)
        L = _lib.lib()
        for t0 in range(0, T, 65535):
            t1 = min(T, t0 + 65535)
            _lib.check(L.tidas_window_frames_f64(_lib.ptr(flat[t0 * n_el:]), t1 - t0, n_el, self.N,
                                                 _lib.ptr(lo_d[t0:]), _lib.ptr(hi_d[t0:]),
                                                 _lib.ptr(first[t0:]), _lib.ptr(last[t0:]),
                                                 _lib.stream_handle()))
        f, l_ = first.cpu().numpy(), last.cpu().numpy()
        has = l_ >= 0
        self.s_lo = np.where(has.any(1), np.where(has, f, np.iinfo(np.int32).max).min(1), 0).astype(np.int64)
        self.s_hi = np.where(has.any(1), l_.max(1) + 1, 0).astype(np.int64)
        self.has_support = has.any(1)


def _next_pow2_vec(n: np.ndarray) -> np.ndarray:
    """1 << bit_length(n - 1), elementwise (frexp gives the exact bit length)."""
    _, e = np.frexp(np.maximum(np.asarray(n, np.int64) - 1, 0).astype(np.float64))
    return np.left_shift(np.int64(1), e.astype(np.int64))


def _cell_geometry(cols, t: int, idx, d_fix: np.ndarray, d_true: np.ndarray):
    """Rebased delays in samples and FFT lengths of the cells (t, every fixed
    profile row of d_fix) — tidas.py:254-265 (offset, span, nfft)."""
    fs = cols.fs
    off = np.minimum(d_fix.min(axis=1), d_true.min())
    df = d_fix - off[:, None]
    dt = d_true[None, :] - off[:, None]
    width = int(cols.s_hi[t] - cols.s_lo[t])
    span = np.ceil(np.maximum(df.max(axis=1), dt.max(axis=1)) * fs).astype(np.int64) + 4
    nfft = _next_pow2_vec(np.maximum(2 * width, width + span))
    return df * fs, dt * fs, nfft


def _theta_from_geometry(cols, idx_of_col, cell_t: np.ndarray, nffts: np.ndarray, dfx_d: torch.Tensor,
                         dtr_d: torch.Tensor, A: int, form: str) -> torch.Tensor:
    """theta of C cells on the device: cell i of column cell_t[i] with FFT length
    nffts[i] and rebased delays dfx_d / dtr_d [C][A] (samples)."""
    dev = _dev()
    L = _lib.lib()
    C = len(cell_t)
    # spectra pairs: distinct (column, nfft)
    keys, cell_pair = np.unique(cell_t.astype(np.int64) * (1 << 32) + nffts, return_inverse=True)
    pair_frame = (keys >> 32).astype(np.int32)
    pair_nfft = (keys & ((1 << 32) - 1)).astype(np.int32)
    P = len(keys)
    kmax = int(pair_nfft.max()) // 2
    rows = np.zeros((P, A), np.int32)
    count = np.zeros(P, np.int32)
    for i in range(P):
        idx = np.asarray(idx_of_col[int(pair_frame[i])], int)
        rows[i, :len(idx)] = idx + cols.n_el // 2  # frame-relative row
        count[i] = len(idx)
    pair_lo = cols.s_lo[pair_frame].astype(np.int32)
    pair_hi = cols.s_hi[pair_frame].astype(np.int32)
    pair_off = np.arange(P, dtype=np.int64) * A
    S = torch.empty((P * A, kmax), dtype=torch.complex128, device=dev)
    keep = [_i32(pair_frame, dev), _i32(pair_lo, dev), _i32(pair_hi, dev), _i32(pair_nfft, dev),
            torch.as_tensor(pair_off).to(dev), _i32(rows, dev), _i32(count, dev)]
    for p0 in range(0, P, 65535):
        p1 = min(P, p0 + 65535)
        _lib.check(L.tidas_window_spectra_f64(
            _lib.ptr(cols.flat), cols.n_el, cols.N, p1 - p0, _lib.ptr(keep[0][p0:]), _lib.ptr(keep[1][p0:]),
            _lib.ptr(keep[2][p0:]), _lib.ptr(keep[3][p0:]), _lib.ptr(keep[4][p0:]), _lib.ptr(keep[5][p0:]),
            A, _lib.ptr(keep[6][p0:]), kmax, _lib.ptr(S), _lib.stream_handle()))
    th_d = torch.empty(C, dtype=torch.float64, device=dev)
    st_d = torch.empty(C, dtype=torch.int32, device=dev)
    cp_d = _i32(cell_pair, dev)
    _lib.check(L.tidas_theta_cells_f64(_lib.ptr(S), C, _lib.ptr(cp_d), _lib.ptr(keep[4]), _lib.ptr(keep[3]),
                                       _lib.ptr(keep[6]), kmax, _lib.ptr(dfx_d), _lib.ptr(dtr_d), A, FORMS[form],
                                       _lib.ptr(th_d), _lib.ptr(st_d), _lib.stream_handle()))
    return th_d


def _good_columns(cols) -> list:
    return [t for t in range(len(cols.ok)) if cols.ok[t] and cols.has_support[t]]


def _theta_cells(cols, idx_of_col, d_fix_of_col, d_true_of_col, form: str) -> np.ndarray:
    """theta [t][r] for every column t and fixed profile row r of d_fix_of_col[t]
    (an (R, n_t) array of delays in seconds) against the column's true profile,
    host geometry (arbitrary profiles: estimate_theta). NaN where the reference
    raises (window outside the frame, no support, zero denominator)."""
    if form not in FORMS:
        raise ValueError(f"unknown estimator form {form!r}")
    dev = _dev()
    T = len(idx_of_col)
    R = d_fix_of_col[0].shape[0]
    theta = np.full((T, R), np.nan)
    good_cols = _good_columns(cols)
    if not good_cols:
        return theta
    A = max(len(idx_of_col[t]) for t in good_cols)
    C = len(good_cols) * R
    dfx = np.zeros((C, A))
    dtr = np.zeros((C, A))
    nffts = np.zeros(C, np.int64)
    cell_t = np.repeat(np.asarray(good_cols, np.int64), R)
    for j, t in enumerate(good_cols):
        n = len(idx_of_col[t])
        df, dt, nf = _cell_geometry(cols, t, idx_of_col[t], d_fix_of_col[t], np.asarray(d_true_of_col[t], float))
        dfx[j * R:(j + 1) * R, :n] = df
        dtr[j * R:(j + 1) * R, :n] = dt
        nffts[j * R:(j + 1) * R] = nf
    th_d = _theta_from_geometry(cols, idx_of_col, cell_t, nffts, _f64(dfx, dev), _f64(dtr, dev), A, form)
    theta[np.asarray(good_cols)] = th_d.cpu().numpy().reshape(len(good_cols), R)
    return theta


def _theta_cells_sweep(cols, halves: np.ndarray, refs: np.ndarray, config: ProbeConfig, form: str) -> np.ndarray:
    """theta [t][r] of a sweep batch: column t's aperture [-halves[t], halves[t]),
    fixed profiles at every reference depth; the cell geometry (delays, FFT
    lengths) is built on the device (tidas_sweep_theta_geometry_f64)."""
    if form not in FORMS:
        raise ValueError(f"unknown estimator form {form!r}")
    dev = _dev()
    L = _lib.lib()
    T, R = len(halves), len(refs)
    theta = np.full((T, R), np.nan)
    good_cols = _good_columns(cols)
    if not good_cols:
        return theta
    A = int(2 * halves[good_cols].max())
    C = len(good_cols) * R
    width = (cols.s_hi - cols.s_lo).astype(np.int32)
    good_d, z_d, h_d, w_d, refs_d = (_i32(good_cols, dev), _f64(cols.targets, dev), _i32(halves, dev),
                                     _i32(width, dev), _f64(refs, dev))
    dfx_d = torch.empty((C, A), dtype=torch.float64, device=dev)
    dtr_d = torch.empty((C, A), dtype=torch.float64, device=dev)
    nfft_d = torch.empty(C, dtype=torch.int32, device=dev)
    _lib.check(L.tidas_sweep_theta_geometry_f64(C, R, _lib.ptr(good_d), _lib.ptr(z_d), _lib.ptr(h_d), _lib.ptr(w_d),
                                                _lib.ptr(refs_d), float(config.pitch), float(config.sound_speed),
                                                float(config.sampling_frequency), A, _lib.ptr(dfx_d),
                                                _lib.ptr(dtr_d), _lib.ptr(nfft_d), _lib.stream_handle()))
    idx_of_col = [np.arange(-int(h), int(h)) for h in halves]
    cell_t = np.repeat(np.asarray(good_cols, np.int64), R)
    th_d = _theta_from_geometry(cols, idx_of_col, cell_t, nfft_d.cpu().numpy().astype(np.int64), dfx_d, dtr_d,
                                A, form)
    theta[np.asarray(good_cols)] = th_d.cpu().numpy().reshape(len(good_cols), R)
    return theta


def _sweep_profiles(cols, halves: np.ndarray, col_d: torch.Tensor, ref_idx_d: torch.Tensor, depths_d: torch.Tensor,
                    config: ProbeConfig, A: int):
    """K3 rows / shifts [C][A] (device) of receive profiles at depths_d[ref_idx_d[c]]
    over column col_d[c]'s aperture, and the cells' crops around the column
    windows (tidas_sweep_crop_geometry_f64). The true-profile PSFs (the column's
    own depth) and the cropped fixed-profile sums share this one device
    expression, so a cell whose reference is its own depth cancels exactly, as
    in the reference's numpy."""
    dev = _dev()
    C = int(col_d.numel())
    h_d = _i32(halves, dev)
    n_d, wlo_d, whi_d = _i32(cols.n_len, dev), _i32(cols.wlo, dev), _i32(cols.whi, dev)
    rows = torch.empty((C, A), dtype=torch.int32, device=dev)
    sh = torch.empty((C, A), dtype=torch.float64, device=dev)
    clo = torch.empty(C, dtype=torch.int32, device=dev)
    chi = torch.empty(C, dtype=torch.int32, device=dev)
    bad = torch.zeros(1, dtype=torch.int32, device=dev)
    _lib.check(_lib.lib().tidas_sweep_crop_geometry_f64(
        C, _lib.ptr(col_d), _lib.ptr(ref_idx_d), _lib.ptr(h_d), _lib.ptr(depths_d), _lib.ptr(wlo_d), _lib.ptr(whi_d),
        _lib.ptr(n_d), cols.n_el, cols.zero_row, cols.N, float(config.pitch), float(config.sound_speed),
        float(config.sampling_frequency), A, _lib.ptr(rows), _lib.ptr(sh), _lib.ptr(clo), _lib.ptr(chi),
        _lib.ptr(bad), _lib.stream_handle()))
    return rows, sh, clo, chi, bad, (h_d, n_d, wlo_d, whi_d)


def theta_matrix_sweep(depth_grid, config: ProbeConfig, tx_rule: ApertureRule, rx_rule: ApertureRule, *,
                       tx_focus_depth: float, window_half_width: float,
                       reference_depths: Optional[np.ndarray] = None, form: str = "beamsum",
                       spreading: bool = True, workers: int = 1):
    """theta for every (reference profile, single-scatterer depth) pair — tidas.py:394-425.

    ``workers`` is accepted for signature compatibility (the GPU batches all cells)."""
    from .tidas import ThetaMatrix
    targets = np.asarray(depth_grid, dtype=float)
    refs = targets if reference_depths is None else np.asarray(reference_depths, dtype=float)
    values = np.full((len(refs), len(targets)), np.nan)
    for b0 in range(0, len(targets), _COL_BATCH):
        tb = targets[b0:b0 + _COL_BATCH]
        cols = _Columns(tb, config, tx_rule, tx_focus_depth, window_half_width, spreading)
        halves = aperture_half_counts(tb, rx_rule, config).astype(np.int64)
        values[:, b0:b0 + len(tb)] = _theta_cells_sweep(cols, halves, refs, config, form).T
        del cols
    return ThetaMatrix(reference_depths=refs, target_depths=targets, values=values)


def error_sweep(depth_grid, config: ProbeConfig, tx_rule: ApertureRule, rx_rule: ApertureRule, *,
                tx_focus_depth: float, window_half_width: float,
                reference_depths: Optional[np.ndarray] = None, form: str = "beamsum",
                spreading: bool = True, delay_method: str = "linear"):
    """(theta, local error, global error) [reference][scatterer depth] matrices of
    run_error_sweep (experiments.py:299-361); the below-5% mask is
    ``np.where(np.isfinite(local), local < 0.05, nan)``."""
    if delay_method != "linear":
        raise NotImplementedError("the GPU error sweep implements delay_method='linear'")
    dev = _dev()
    L = _lib.lib()
    targets = np.asarray(depth_grid, dtype=float)
    refs = targets if reference_depths is None else np.asarray(reference_depths, dtype=float)
    R, T = len(refs), len(targets)
    th_m, loc_m, glo_m = (np.full((R, T), np.nan) for _ in range(3))
    refs_d = _f64(refs, dev)
    for b0 in range(0, T, _COL_BATCH):
        tb = targets[b0:b0 + _COL_BATCH]
        cols = _Columns(tb, config, tx_rule, tx_focus_depth, window_half_width, spreading)
        halves = aperture_half_counts(tb, rx_rule, config).astype(np.int64)
        A = int(2 * halves.max())
        # true-profile PSF per column (das_psf of the windowed frame), K3
        cols_d = torch.arange(len(tb), dtype=torch.int32, device=dev)
        z_d = _f64(tb, dev)
        rows_t, sh_t, _, _, bad_t, _ = _sweep_profiles(cols, halves, cols_d, cols_d, z_d, config, A)
        _das._count(int(2 * halves.sum()))
        psf_d = _das._delayed_sums_dev(cols.flat, rows_t, sh_t)
        th = _theta_cells_sweep(cols, halves, refs, config, form)  # [t][r]
        th_m[:, b0:b0 + len(tb)] = th.T
        t_sel, r_sel = np.nonzero(np.isfinite(th))
        C = t_sel.size
        if C == 0:
            continue
        # fixed-profile sums on each cell's crop [lo - span, hi + 2) (tidas.py:336-349), K3
        cc_d, cr_d = _i32(t_sel, dev), _i32(r_sel, dev)
        rows_c, sh_c, clo_d, chi_d, bad, (_, n_d, wlo_d, whi_d) = _sweep_profiles(
            cols, halves, cc_d, cr_d, refs_d, config, A)
        _das._count(int((2 * halves)[t_sel].sum()))
        sums = _das._delayed_sums_dev(cols.flat, rows_c, sh_c, lo=clo_d, hi=chi_d)
        th_d = _f64(th[t_sel, r_sel], dev)
        out = torch.empty((C, 4), dtype=torch.float64, device=dev)
        _lib.check(L.tidas_psf_errors_f64(_lib.ptr(sums), cols.N, _lib.ptr(th_d), _lib.ptr(psf_d), C,
                                          _lib.ptr(cc_d), _lib.ptr(clo_d), _lib.ptr(chi_d), _lib.ptr(n_d),
                                          _lib.ptr(wlo_d), _lib.ptr(whi_d), _lib.ptr(out), _lib.stream_handle()))
        if int(bad.item()) or int(bad_t.item()):
            raise ValueError(f"a fixed-profile delay shift exceeds the trace support {cols.N}")
        e = out.cpu().numpy()
        with np.errstate(divide="ignore", invalid="ignore"):
            loc = np.where(e[:, 1] > 0.0, e[:, 0] / np.where(e[:, 1] > 0.0, e[:, 1], 1.0), np.nan)
            glo = np.where(e[:, 3] > 0.0, e[:, 2] / np.where(e[:, 3] > 0.0, e[:, 3], 1.0), np.nan)
        # a failing local_error (experiments.py:327) leaves the global error unset
        glo = np.where(np.isfinite(loc), glo, np.nan)
        loc_m[r_sel, b0 + t_sel] = loc
        glo_m[r_sel, b0 + t_sel] = glo
        del cols, sums, psf_d
    return th_m, loc_m, glo_m


def estimate_theta(windowed_frame: RfFrame, fixed_delays: DelayProfile, true_delays: DelayProfile,
                   form: str = "beamsum", support: Optional[Tuple[int, int]] = None) -> float:
    """Least-squares scaling weight over the window spectrum — tidas.py:237-283."""
    if len(fixed_delays) != len(true_delays) or np.any(
            np.asarray(fixed_delays.element_indices) != np.asarray(true_delays.element_indices)):
        raise ValueError("fixed and true profiles must cover the same aperture")
    if form not in FORMS:
        raise ValueError(f"unknown estimator form {form!r}")
    dev = _dev()
    L = _lib.lib()
    tr = np.asarray(windowed_frame.traces, float)
    n_el, n = tr.shape
    lo, hi = (0, n) if support is None else (int(support[0]), int(support[1]))

    class _One:  # a one-column stand-in for _Columns
        pass

    one = _One()
    one.fs, one.n_el, one.N = windowed_frame.sampling_frequency, n_el, n
    one.flat = _f64(tr, dev)
    first = torch.empty((1, n_el), dtype=torch.int32, device=dev)
    last = torch.empty((1, n_el), dtype=torch.int32, device=dev)
    scan = one.flat.clone()  # the scan zeroes outside [lo, hi): keep the caller's samples
    lo_d, hi_d = _i32([lo], dev), _i32([hi], dev)  # alive until the launch is enqueued
    _lib.check(L.tidas_window_frames_f64(_lib.ptr(scan), 1, n_el, n, _lib.ptr(lo_d), _lib.ptr(hi_d),
                                         _lib.ptr(first), _lib.ptr(last), _lib.stream_handle()))
    f, l_ = first.cpu().numpy()[0], last.cpu().numpy()[0]
    if not (l_ >= 0).any():
        raise ZeroDivisionError("window missed the echo: frame is zero inside the window")
    one.s_lo = np.array([f[l_ >= 0].min()])
    one.s_hi = np.array([l_.max() + 1])
    one.ok = np.array([True])
    one.has_support = np.array([True])
    idx = np.asarray(fixed_delays.element_indices, int)
    th = _theta_cells(one, [idx], [np.asarray(fixed_delays.delays, float)[None, :]],
                      [np.asarray(true_delays.delays, float)], form)
    if not np.isfinite(th[0, 0]):
        raise ZeroDivisionError("window missed the echo: fixed-profile sum has no energy")
    return float(th[0, 0])
