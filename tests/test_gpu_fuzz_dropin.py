"""Seeded randomised cases through the drop-in reference API (the reference's
pkg/src/tidas surface, FP64) against the oracle restatement.

Random probes (element counts, pitches, sampling rates), random RF frames with
t0 >= 0 and a random focused-transmit aperture, random depth grids, the three
aperture rules, optional envelope windows, on- and off-axis pixels:

* das_line / das_value — the three internal paths (analytic gather when the
  traces have zero heads / tails, full-trace delayed sums otherwise, the
  windowed K3 + K4 path) against das_value_fulltrace (das.py:181-193) and the
  windowed envelope read (das.py:174-178);
* tidas_line (tidas.py:493-531) with random fixed profiles and thetas;
* estimate_theta_aligned (tidas.py:286-314) with random true profiles.

Tolerance: 1e-10 of the line's largest value (FP64 throughout; the golden
vectors of test_gpu_dropin.py are matched at 1e-12).
"""
import os

import numpy as np
import pytest

import paper_2507_15464_b200 as T
from oracle import das as od
from oracle import geom
from oracle import tidas as ot

pytestmark = pytest.mark.gpu
N_SEEDS = int(os.environ.get("TIDAS_FUZZ_SEEDS", "24"))
TOL = 1e-10


def _rule(rng):
    k = int(rng.integers(0, 3))
    if k == 0:
        f = float(rng.uniform(0.5, 3.0))
        return T.FNumber(f), ("fnumber", f)
    if k == 1:
        n = int(rng.integers(1, 40))
        return T.FixedCount(n), ("fixed", n)
    kk = float(rng.uniform(0.2, 1.0))
    return T.Kossoff(kk), ("kossoff", kk)


def _case(seed):
    rng = np.random.default_rng(20000 + seed)
    n_el = int(rng.choice([8, 16, 32, 64, 96]))
    f0 = float(rng.uniform(2e6, 8e6))
    fs = float(rng.choice([4.0, 5.0, 6.25, 8.0])) * f0 * float(rng.uniform(1.0, 1.5))
    probe = T.ProbeConfig(element_count=n_el, pitch=float(rng.uniform(0.1e-3, 0.4e-3)), center_frequency=f0,
                          sampling_frequency=fs, sound_speed=1540.0)
    c = probe.sound_speed
    n = int(rng.integers(600, 3000))
    t0 = float(rng.choice([0.0, 0.0, rng.uniform(0, 200) / fs]))
    traces = rng.standard_normal((n_el, n))
    if rng.random() < 0.5:  # zero heads / tails: the exact analytic-gather path
        head, tail = int(rng.integers(0, n // 4)), int(rng.integers(0, n // 4))
        traces[:, :head] = 0.0
        traces[:, n - tail:] = 0.0
    tx_half = int(rng.integers(1, n_el // 2 + 1))
    tx_idx = np.arange(-tx_half, tx_half)
    frame = T.RfFrame(traces=traces, sampling_frequency=fs, t0=t0,
                      tx_focus_depth=float(rng.uniform(5e-3, 40e-3)), aperture=tx_idx)
    # depths inside the trace: two-way travel <= ~0.9 of the trace, clear of the
    # receive shifts reaching past the row
    z_hi = 0.45 * (t0 + (n - 1) / fs) * c
    nz = int(rng.integers(1, 24))
    z = np.sort(rng.uniform(0.15 * z_hi, z_hi, nz))
    z = z[np.concatenate([[True], np.diff(z) > 0])]
    rule, orule = _rule(rng)
    half_width = None if rng.random() < 0.5 else float(rng.uniform(3, 60)) / fs
    return probe, frame, z, rule, orule, half_width, rng


def _oracle_pixel(frame, probe, x, z, orule, half_width):
    fs, c, pitch = frame.sampling_frequency, probe.sound_speed, probe.pitch
    h = geom.ref_aperture_half(z, orule, probe.element_count, pitch, probe.wavelength)
    tx_xs = (np.asarray(frame.aperture) + 0.5) * pitch
    t_star = float(geom.focused_tx_arrival(x, z, frame.tx_focus_depth, tx_xs, c)) + z / c
    if half_width is None:
        return od.das_value_fulltrace(frame.traces, fs, frame.t0, x, z, h, pitch, c, t_star)
    idx = np.arange(-h, h)
    delays = geom.receive_delays(x, z, (idx + 0.5) * pitch, c)
    summed = od.delayed_sum(frame.traces, fs, idx, delays)
    return ot.windowed_envelope_value(summed, fs, frame.t0, t_star, half_width)


def _close(got, ref, what):
    got, ref = np.asarray(got, float), np.asarray(ref, float)
    scale = max(float(np.max(np.abs(ref))) if ref.size else 0.0, 1e-300)
    assert float(np.max(np.abs(got - ref))) <= TOL * scale, (what, float(np.max(np.abs(got - ref))) / scale)


def _shifts_fit(frame, probe, xs, zs, orule):
    """The reference raises when a receive shift reaches the trace length."""
    for x, z in zip(xs, zs):
        h = geom.ref_aperture_half(z, orule, probe.element_count, probe.pitch, probe.wavelength)
        d = geom.receive_delays(x, z, (np.arange(-h, h) + 0.5) * probe.pitch, probe.sound_speed)
        if np.max(np.abs(d)) * frame.sampling_frequency >= frame.n_samples:
            return False
    return True


@pytest.mark.parametrize("seed", range(N_SEEDS))
def test_das_line_random_frames_vs_oracle(seed):
    probe, frame, z, rule, orule, hw, _ = _case(seed)
    if not _shifts_fit(frame, probe, np.zeros_like(z), z, orule):
        with pytest.raises(ValueError):
            T.das_line(frame, z, probe, rule, envelope_half_width=hw)
        return
    line = T.das_line(frame, z, probe, rule, envelope_half_width=hw)
    ref = [_oracle_pixel(frame, probe, 0.0, zz, orule, hw) for zz in z]
    _close(line, ref, ("das_line", seed, hw is not None))


@pytest.mark.parametrize("seed", range(N_SEEDS))
def test_das_value_off_axis_random_frames_vs_oracle(seed):
    probe, frame, z, rule, orule, hw, rng = _case(seed)
    xs = rng.uniform(-0.5, 0.5, len(z)) * probe.element_count * probe.pitch
    if not _shifts_fit(frame, probe, xs, z, orule):
        return
    got = [T.das_value(frame, (float(x), float(zz)), probe, rule, envelope_half_width=hw) for x, zz in zip(xs, z)]
    ref = [_oracle_pixel(frame, probe, float(x), float(zz), orule, hw) for x, zz in zip(xs, z)]
    _close(got, ref, ("das_value", seed))


@pytest.mark.parametrize("seed", range(N_SEEDS))
def test_tidas_line_and_theta_random_profiles_vs_oracle(seed):
    probe, frame, z, rule, orule, hw, rng = _case(seed)
    fs, c, pitch = frame.sampling_frequency, probe.sound_speed, probe.pitch
    hw = hw if hw is not None else float(rng.uniform(3, 60)) / fs
    h = int(rng.integers(1, probe.element_count // 2 + 1))
    fixed = T.rx_delay_profile(float(rng.uniform(0.3, 1.0)) * z[-1], np.arange(-h, h), probe)
    if np.max(np.abs(fixed.delays)) * fs >= frame.n_samples:
        return
    thetas = rng.uniform(0.2, 3.0, len(z))
    line = T.tidas_line(frame, fixed, thetas, z, probe, window_half_width=hw)
    tx_xs = (np.asarray(frame.aperture) + 0.5) * pitch
    t_stars = geom.focused_tx_arrival(np.zeros_like(z), z, frame.tx_focus_depth, tx_xs, c) + z / c
    ref = ot.tidas_line(frame.traces, fs, frame.t0, fixed.element_indices, fixed.delays, thetas, t_stars, hw)
    _close(line, ref, ("tidas_line", seed))
    # theta of a random true profile over a window around one depth
    true = T.rx_delay_profile(float(z[0]), np.arange(-h, h), probe)
    win = T.TimeWindow(center=float(t_stars[0]), half_width=hw)
    try:
        ref_t = ot.estimate_theta_aligned(frame.traces, fs, frame.t0, win.center, hw, fixed.element_indices,
                                          fixed.delays, true.element_indices, true.delays)
    except (ValueError, ZeroDivisionError) as e:
        with pytest.raises(type(e)):
            T.estimate_theta_aligned(frame, win, fixed, true)
        return
    got_t = T.estimate_theta_aligned(frame, win, fixed, true)
    assert abs(got_t - ref_t) <= TOL * max(abs(ref_t), 1.0), (seed, got_t, ref_t)
