"""Drop-in for the reference's ``tidas.das`` (pkg/src/tidas/das.py:17-28).

Same names, signatures, return types and exceptions; the numerical loops run
in the CUDA library in float64:

* ``delayed_sum`` / ``apply_fractional_delay`` / ``das_psf`` -> K3
  ``tidas_delayed_sum_f64`` (bit-identical to the numpy reference);
* ``das_value`` / ``das_line`` -> K1 analytic RF + K2 ``tidas_das_image``
  (O(channels) per pixel analytic gather), or — when a
  channel lacks the leading zeros that make the gather exact — the full-trace
  GPU path K3 + K1 (envelope) + interpolation, like the reference;
* windowed envelopes (``envelope_half_width``) -> K3 restricted to the window +
  K4 ``tidas_window_envelope_f64``.

The instrumentation counter ``_delay_ops`` (das.py:30-41) counts fractional-delay
applications exactly as the reference does.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Tuple

import numpy as np
import torch

from . import _lib
from . import imaging
from .geometry import ApertureRule, ProbeConfig, aperture_half_counts, element_positions, rx_aperture
from .simulate import RfFrame, tx_arrival_time, _focused_arrivals

__all__ = ["Trace", "apply_fractional_delay", "delayed_sum", "das_psf", "das_value", "das_line",
           "expected_arrival_time", "target_delays", "reset_delay_counter", "delay_counter"]

_delay_ops = 0


def reset_delay_counter() -> None:
    global _delay_ops
    _delay_ops = 0


def delay_counter() -> int:
    return _delay_ops


def _count(n: int) -> None:
    global _delay_ops
    _delay_ops += int(n)


@dataclass
class Trace:
    """One time signal on a uniform grid starting at t0."""

    samples: np.ndarray
    sampling_frequency: float
    t0: float = 0.0

    def __post_init__(self) -> None:
        self.samples = np.asarray(self.samples)
        if self.samples.ndim != 1 or len(self.samples) < 1:
            raise ValueError("trace needs a 1-D, non-empty sample array")

    @property
    def duration(self) -> float:
        return len(self.samples) / self.sampling_frequency

    @property
    def times(self) -> np.ndarray:
        return self.t0 + np.arange(len(self.samples)) / self.sampling_frequency

    def __len__(self) -> int:
        return len(self.samples)


def _device():
    return torch.device("cuda", torch.cuda.current_device())


def _to_dev(a, dtype=torch.float64):
    return torch.as_tensor(np.ascontiguousarray(a)).to(device=_device(), dtype=dtype)


def _check_shifts(shifts: np.ndarray, n: int) -> None:
    # das.py:87-88: |delay| * fs >= n is rejected
    if shifts.size and np.max(np.abs(shifts)) >= n:
        bad = float(shifts.flat[int(np.argmax(np.abs(shifts)))])
        raise ValueError(f"delay shift {bad} samples exceeds the trace support {n}")


def _delayed_sums_dev(traces_d: torch.Tensor, rows: np.ndarray, shifts: np.ndarray,
                      lo: Optional[np.ndarray] = None, hi: Optional[np.ndarray] = None,
                      out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """K3 over P profiles: rows/shifts [P][T] -> [P][N] float64 on the device.
    rows / shifts / lo / hi are host arrays, or device tensors (int32 / float64 /
    int32 / int32) whose builder has checked the shifts (the sweep's crop geometry)."""
    L = _lib.lib()
    P, T = rows.shape
    n_rows, N = traces_d.shape
    if out is None:
        out = torch.zeros((P, N), dtype=torch.float64, device=traces_d.device)
    if isinstance(rows, torch.Tensor):
        r_d, s_d, lo_d, hi_d = rows, shifts, lo, hi
    else:
        _check_shifts(shifts, N)
        r_d = _to_dev(rows.astype(np.int32), torch.int32)
        s_d = _to_dev(shifts.astype(np.float64))
        lo_d = _to_dev(lo.astype(np.int32), torch.int32) if lo is not None else None
        hi_d = _to_dev(hi.astype(np.int32), torch.int32) if hi is not None else None
    for p0 in range(0, P, 65535):
        p1 = min(P, p0 + 65535)
        _lib.check(L.tidas_delayed_sum_f64(
            _lib.ptr(traces_d), n_rows, N, _lib.ptr(r_d[p0:p1]), _lib.ptr(s_d[p0:p1]), T, p1 - p0,
            _lib.ptr(lo_d[p0:p1]) if lo_d is not None else None,
            _lib.ptr(hi_d[p0:p1]) if hi_d is not None else None,
            _lib.ptr(out[p0:p1]), _lib.stream_handle()))
    return out


def apply_fractional_delay(trace: Trace, delay: float, method: str = "linear") -> Trace:
    """out(t) = in(t - delay) — das.py:115-123 (linear: K3; spectral: DFT phase ramp)."""
    _count(1)
    n = len(trace.samples)
    if abs(delay) * trace.sampling_frequency >= n:
        raise ValueError(f"delay {delay} s exceeds the trace support {n / trace.sampling_frequency} s")
    shift = delay * trace.sampling_frequency
    if method == "linear":
        x = _to_dev(np.asarray(trace.samples, float)[None, :])
        out = _delayed_sums_dev(x, np.zeros((1, 1), np.int32), np.array([[shift]]))
        return Trace(out[0].cpu().numpy(), trace.sampling_frequency, trace.t0)
    if method == "spectral":
        from .metrics import spectral_delay
        return Trace(spectral_delay(np.asarray(trace.samples, float), shift),
                     trace.sampling_frequency, trace.t0)
    raise ValueError(f"unknown delay method {method!r}")


def target_delays(target: Tuple[float, float], aperture, config: ProbeConfig) -> np.ndarray:
    """(z - hypot(x - x_n, z)) / c — das.py:126-132."""
    x, z = target
    xs = element_positions(np.asarray(aperture), config)
    return (z - np.hypot(x - xs, z)) / config.sound_speed


def expected_arrival_time(target: Tuple[float, float], frame: RfFrame, config: ProbeConfig) -> float:
    return tx_arrival_time(target, frame.tx_focus_depth, frame.aperture, config) + target[1] / config.sound_speed


def delayed_sum(frame: RfFrame, element_indices, delays, method: str = "linear") -> Trace:
    """Sum of shifted traces in aperture order — das.py:140-149 (K3, bit-identical)."""
    fs = frame.sampling_frequency
    idx = np.asarray(element_indices).astype(np.int64)
    d = np.asarray(delays, dtype=float)
    if method != "linear":
        if method != "spectral":
            raise ValueError(f"unknown delay method {method!r}")
        total = np.zeros(frame.n_samples)
        for i, dl in zip(idx, d):
            total += apply_fractional_delay(Trace(frame.traces[frame.row(i)], fs), dl, method).samples
        return Trace(total, fs, frame.t0)
    _count(len(idx))
    half = frame.traces.shape[0] // 2
    rows = (idx + half)[None, :]
    x = _to_dev(np.asarray(frame.traces, float))
    out = _delayed_sums_dev(x, rows, (d * fs)[None, :])
    return Trace(out[0].cpu().numpy(), fs, frame.t0)


def das_psf(frame: RfFrame, target: Tuple[float, float], config: ProbeConfig,
            rx_rule: ApertureRule, method: str = "linear") -> Trace:
    aperture = rx_aperture(target[1], rx_rule, config)
    return delayed_sum(frame, aperture, target_delays(target, aperture, config), method)


# ------------------------------------------------------------------ pixels


def _window_bounds_arr(n, t0, fs, centers, half_width):
    lo = np.ceil((np.asarray(centers) - half_width - t0) * fs - 1e-9).astype(np.int64)
    hi = np.floor((np.asarray(centers) + half_width - t0) * fs + 1e-9).astype(np.int64)
    return np.maximum(lo, 0), np.minimum(hi, n - 1) + 1


def _pixels(frame: RfFrame, xs: np.ndarray, zs: np.ndarray, config: ProbeConfig,
            rx_rule: ApertureRule, envelope_half_width: Optional[float]) -> np.ndarray:
    """DAS values of pixels (xs[p], zs[p]) of one frame, reference semantics.

    Host geometry is vectorised over the pixels (the same float operations as
    rx_aperture / target_delays per pixel, das.py:126-132, geometry.py:188-199)."""
    fs, c, t0 = frame.sampling_frequency, config.sound_speed, frame.t0
    n_el, N = frame.traces.shape
    half = n_el // 2
    P = len(zs)
    t_star = _focused_arrivals(xs, zs, frame.tx_focus_depth, frame.aperture, config) + zs / c
    ap_half = aperture_half_counts(zs, rx_rule, config).astype(np.int32)
    _count(int(np.sum(2 * ap_half)))
    # per-pixel receive shifts [P][T] over the array-centred aperture, padded taps
    # (beyond 2 * ap_half) point at a real row with shift 0 and are masked out
    T = int(2 * ap_half.max())
    j = np.arange(T)[None, :]
    live = j < 2 * ap_half[:, None]
    idx = np.where(live, j - ap_half[:, None], 0)
    el_x = (idx + 0.5) * config.pitch
    shifts = np.where(live, (zs[:, None] - np.hypot(xs[:, None] - el_x, zs[:, None])) / c * fs, 0.0)
    rows = (idx + half).astype(np.int64)
    _check_shifts(shifts, N)
    x_d = _to_dev(np.asarray(frame.traces, float))
    if envelope_half_width is not None:
        lo, hi = _window_bounds_arr(N, t0, fs, t_star, envelope_half_width)
        out = torch.zeros((P, N), dtype=torch.float64, device=x_d.device)
        # run the exact-length profiles separately (padding taps would add 0 * x)
        for T_p in np.unique(2 * ap_half):
            sel = np.flatnonzero(2 * ap_half == T_p)
            sub = _delayed_sums_dev(x_d, rows[sel, :T_p], shifts[sel, :T_p],
                                    lo[sel], np.maximum(hi[sel], lo[sel]))
            out[torch.as_tensor(sel, device=x_d.device)] = sub
        return _window_read(out, lo, hi, (t_star - t0) * fs, None)
    # exact analytic gather needs zero-fill == circular shift on every used channel
    support = torch.empty((n_el, 2), dtype=torch.int32, device=x_d.device)
    A = imaging.rf_analytic(x_d, "f64", support=support)
    if _gather_exact(support.cpu().numpy(), rows, shifts, 2 * ap_half, N) and np.all(xs == xs[0]):
        plan = imaging.table_plan(n_el=n_el, pitch=config.pitch, fs=fs, c=c, n_samples=N,
                                  x=xs[:1], z=zs, t_star=t_star[None, :, None],
                                  aperture=("ref", ap_half), out="envelope", prec="f64", t0=t0)
        img = imaging.das_from_analytic(A.view(1, 1, n_el, N), plan)
        return img[0, :, 0].cpu().numpy()
    # full-trace path (reference algorithm on the GPU)
    out = torch.zeros((P, N), dtype=torch.float64, device=x_d.device)
    for T_p in np.unique(2 * ap_half):
        sel = np.flatnonzero(2 * ap_half == T_p)
        out[torch.as_tensor(sel, device=x_d.device)] = _delayed_sums_dev(x_d, rows[sel, :T_p], shifts[sel, :T_p])
    env = imaging.rf_analytic(out, "f64").abs()
    return _interp_rows(env, (t_star - t0) * fs)


def _gather_exact(sup: np.ndarray, rows: np.ndarray, shifts: np.ndarray, counts, N: int) -> bool:
    """SURVEY Appendix B.1 precondition: for every used channel with shift s,
    m = floor/ceil(s): m < 0 needs first_nonzero >= -m (no wrapped head sample),
    m >= 0 needs last_nonzero <= N - m - 2 (no wrapped tail sample)."""
    used = np.arange(rows.shape[1])[None, :] < np.asarray(counts)[:, None]
    first, last = sup[rows, 0], sup[rows, 1]
    live = used & (first >= 0)
    mlo, mhi = np.floor(shifts), np.ceil(shifts)
    if np.any(live & (mlo < 0) & (first < -mlo)):
        return False
    return not np.any(live & (mhi >= 0) & (last > N - mhi - 2))


def _interp_rows(env: torch.Tensor, pos: np.ndarray) -> np.ndarray:
    """np.interp(pos_p, arange(N), env[p], left=0, right=0) per row."""
    e = env.cpu().numpy()
    N = e.shape[1]
    out = np.zeros(len(pos))
    for p, q in enumerate(pos):
        out[p] = float(np.interp(q, np.arange(N), e[p], left=0.0, right=0.0))
    return out


def _window_read(traces_d: torch.Tensor, lo, hi, pos, theta) -> np.ndarray:
    """K4 over P pixels, pixel p reading row p of traces_d."""
    L = _lib.lib()
    P, N = traces_d.shape
    out = torch.empty(P, dtype=torch.float64, device=traces_d.device)
    # keep every argument tensor referenced until the launch is enqueued: a
    # temporary freed earlier would be handed to the next allocation
    tr = _to_dev(np.arange(P, dtype=np.int32), torch.int32)
    th = _to_dev(np.asarray(theta, float)) if theta is not None else None
    lo_d = _to_dev(np.asarray(lo, np.int32), torch.int32)
    hi_d = _to_dev(np.asarray(hi, np.int32), torch.int32)
    pos_d = _to_dev(np.asarray(pos, float))
    _lib.check(L.tidas_window_envelope_f64(
        _lib.ptr(traces_d), N, _lib.ptr(tr), _lib.ptr(lo_d), _lib.ptr(hi_d), _lib.ptr(pos_d),
        _lib.ptr(th), P, _lib.ptr(out), _lib.stream_handle()))
    return out.cpu().numpy()


def das_value(frame: RfFrame, target: Tuple[float, float], config: ProbeConfig,
              rx_rule: ApertureRule, *, envelope_half_width: Optional[float] = None,
              method: str = "linear") -> float:
    """PSF envelope at the expected arrival of ``target`` — das.py:181-193."""
    if method != "linear":
        from .metrics import envelope, window_bounds  # spectral: reference composition
        psf = das_psf(frame, target, config, rx_rule, method)
        t = expected_arrival_time(target, frame, config)
        return _envelope_at_host(psf, t, envelope_half_width)
    x, z = target
    if z <= 0:
        raise ValueError(f"depth must be positive, got {z}")
    return float(_pixels(frame, np.array([float(x)]), np.array([float(z)]), config, rx_rule,
                         envelope_half_width)[0])


def _envelope_at_host(psf: Trace, t: float, half_width):
    from .metrics import envelope, window_bounds
    fs = psf.sampling_frequency
    pos = (t - psf.t0) * fs
    if half_width is None:
        env = envelope(psf).samples
        return float(np.interp(pos, np.arange(len(env)), env, left=0.0, right=0.0))
    lo, hi = window_bounds(len(psf.samples), psf.t0, fs, t, half_width)
    if hi - lo < 4:
        return 0.0
    env = envelope(Trace(psf.samples[lo:hi], fs, 0.0)).samples
    return float(np.interp(pos - lo, np.arange(len(env)), env, left=0.0, right=0.0))


def das_line(frame: RfFrame, depths, config: ProbeConfig, rx_rule: ApertureRule, *,
             envelope_half_width: Optional[float] = None, method: str = "linear") -> np.ndarray:
    """Central-line dynamic-focus reconstruction — das.py:196-221."""
    depths = np.asarray(depths, dtype=float)
    if np.any(np.diff(depths) <= 0) or np.any(depths <= 0):
        raise ValueError("depths must be strictly increasing and positive")
    if method != "linear":
        return np.array([das_value(frame, (0.0, z), config, rx_rule,
                                   envelope_half_width=envelope_half_width, method=method)
                         for z in depths])
    if len(depths) == 0:
        return np.zeros(0)
    return _pixels(frame, np.zeros_like(depths), depths, config, rx_rule, envelope_half_width)
