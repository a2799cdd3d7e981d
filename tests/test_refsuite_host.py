"""The reference's own unit tests, restated against the drop-in — host-side part.

The reference suite (/root/reference/pkg/tests) cannot travel to the GPU box and
is not copied here; each test below re-asserts, on the drop-in package, the
property one reference test checks (same inputs, same tolerance), citing it as
``ref: <file>:<line>``. This file holds the cases that need no device
(geometry, host metrics, containers, persistence); tests/test_gpu_refsuite.py
holds the rest. Not restated (out of scope, SURVEY §8 / DESIGN §9): test_cli.py,
test_experiments.py, test_acceptance.py, and test_tidas.py:321 (DepthGrid, an
experiments.py type).
"""
import json

import numpy as np
import pytest

import paper_2507_15464_b200 as T
from paper_2507_15464_b200.metrics import DB_FLOOR, width_at_half_max, window_bounds, write_reports

FS = 50e6


@pytest.fixture(scope="module")
def probe():
    return T.ProbeConfig()


def burst(sigma=40.0, n=512, carrier=0.14, amp=1.0):
    k = np.arange(n)
    env = amp * np.exp(-((k - n / 2) ** 2) / (2 * sigma ** 2))
    return env * np.sin(2 * np.pi * carrier * k), env


# ------------------------------------------------------------ test_geometry.py


def test_probe_defaults(probe):  # ref: test_geometry.py:21
    assert probe.element_count == 192
    assert probe.wavelength == pytest.approx(1540.0 / 7e6)


@pytest.mark.parametrize("bad", [dict(element_count=3), dict(element_count=0), dict(pitch=0.0),
                                 dict(sound_speed=-1.0), dict(sampling_frequency=20e6)])
def test_probe_invariants(bad):  # ref: test_geometry.py:35
    with pytest.raises(ValueError):
        T.ProbeConfig(**bad)


def test_probe_json(probe, tmp_path):  # ref: test_geometry.py:39
    p = tmp_path / "probe.json"
    probe.to_json(p)
    assert T.ProbeConfig.from_json(p) == probe
    assert set(json.loads(p.read_text())) == {"element_count", "pitch", "center_frequency",
                                               "sampling_frequency", "sound_speed", "pulse_cycles",
                                               "fractional_bandwidth"}


def test_element_positions(probe):  # ref: test_geometry.py:58, :62, :66, :72
    assert T.element_position(-1, probe) == pytest.approx(-0.1e-3)
    assert T.element_position(0, probe) == pytest.approx(0.1e-3)
    assert T.element_position(95, probe) == pytest.approx(19.1e-3)
    for n in (96, -97):
        with pytest.raises(ValueError):
            T.element_position(n, probe)
    xs = T.element_positions(np.arange(-96, 96), probe)
    assert np.all(xs != 0.0) and np.allclose(np.sort(xs) + np.sort(xs)[::-1], 0.0)


def test_rx_delay_hand_value():  # ref: test_geometry.py:79
    prof = T.rx_delay_profile(25e-3, np.array([49]), T.ProbeConfig(pitch=10e-3 / 49.5))
    assert prof.delays[0] == pytest.approx(-1.250535088e-6, rel=1e-8)


def test_rx_delay_shape_properties(probe):  # ref: test_geometry.py:87, :91, :95, :118
    d = T.rx_delay_profile(17e-3, np.arange(-96, 96), probe).delays
    assert np.array_equal(d, d[::-1])
    assert np.all(T.rx_delay_profile(5e-3, np.arange(-96, 96), probe).delays <= 0.0)
    mags = [abs(T.rx_delay_profile(z, np.array([40]), probe).delays[0]) for z in np.linspace(5e-3, 60e-3, 24)]
    assert np.all(np.diff(mags) < 0.0)
    with pytest.raises(ValueError):
        T.rx_delay_profile(0.0, np.arange(-2, 2), probe)


def test_rx_delay_taylor_remainder(probe):  # ref: test_geometry.py:100
    z0, x, c = 25e-3, T.element_position(60, probe), probe.sound_speed
    D = lambda z: T.rx_delay_profile(z, np.array([60]), probe).delays[0]  # noqa: E731
    slope = (1.0 - z0 / np.hypot(x, z0)) / c
    curv = x * x / np.hypot(x, z0) ** 3 / c
    for dz in np.linspace(-2e-3, 2e-3, 41):
        if dz != 0.0:
            assert abs(D(z0 + dz) - D(z0) - slope * dz) <= 1.2 * curv * dz * dz


def test_delay_relative_variation(probe):  # ref: test_geometry.py:124, :127, :132
    assert T.delay_relative_variation(10, 25e-3, 25e-3, probe) == 0.0
    assert T.delay_relative_variation(0, 25e-3, 26e-3, probe) == pytest.approx(-0.04, abs=1e-6)
    v = [abs(T.delay_relative_variation(n, 25e-3, 26e-3, probe)) for n in range(0, 96, 5)]
    assert np.all(np.diff(v) < 0.0)


def test_apertures(probe):  # ref: test_geometry.py:138-176
    ap = T.rx_aperture(19.2e-3, T.FNumber(1.0), probe)
    assert len(ap) == 96 and ap[0] == -48 and ap[-1] == 47
    assert len(T.rx_aperture(38.4e-3, T.FNumber(1.0), probe)) == 192
    assert len(T.rx_aperture(60e-3, T.FNumber(1.0), probe)) == 192
    assert len(T.rx_aperture(1e-6, T.FNumber(1.0), probe)) == 2
    w = [len(T.rx_aperture(z, T.FNumber(1.0), probe)) for z in np.linspace(1e-3, 50e-3, 80)]
    assert np.all(np.diff(w) >= 0) and w[-1] == 192
    assert len(T.tx_aperture(25e-3, T.Kossoff(0.6), probe)) == 30
    assert len(T.tx_aperture(25e-3, T.Kossoff(1.0), probe)) == 22
    for z in (5e-3, 25e-3, 45e-3):
        ap = T.tx_aperture(z, T.FixedCount(64), probe)
        assert len(ap) == 64 and ap[0] == -32
    for bad in (lambda: T.FNumber(0.0), lambda: T.FixedCount(0), lambda: T.Kossoff(1.5)):
        with pytest.raises(ValueError):
            bad()
    for z in (3e-3, 11e-3, 33e-3):  # ref: test_geometry.py:178
        ap = T.rx_aperture(z, T.FNumber(1.0), probe)
        assert np.array_equal(ap, np.arange(-len(ap) // 2, len(ap) // 2))


# --------------------------------------------------- test_metrics.py (host)


def test_width_at_half_max_shapes():  # ref: test_metrics.py:48, :55, :61, :68
    tri = np.concatenate([np.linspace(0, 5.0, 100), np.linspace(5.0, 0, 100)])
    assert width_at_half_max(tri, FS) == pytest.approx(99 / FS, rel=0.02)
    rect = np.zeros(100)
    rect[30:70] = 1.0
    assert width_at_half_max(rect, FS) == pytest.approx(40 / FS, rel=0.05)
    k = np.arange(600)
    g = np.exp(-((k - 300) ** 2) / (2 * 25.0 ** 2))
    assert width_at_half_max(g, FS) == pytest.approx(2 * np.sqrt(2 * np.log(2)) * 25 / FS, rel=1e-3)
    with pytest.raises(ValueError):
        width_at_half_max(np.ones(50), FS)


def test_error_metrics():  # ref: test_metrics.py:88, :95, :104, :108, :116, :122
    x, _ = burst()
    t = T.Trace(x, FS)
    w = T.TimeWindow(256 / FS, 64 / FS)
    assert T.local_error(t, t, w) == 0.0 and T.global_error(t, t) == 0.0
    cand = T.Trace(1.07 * x, FS)
    w2 = T.TimeWindow(256 / FS, 100 / FS)
    assert T.local_error(t, cand, w2) == pytest.approx(0.07 ** 2, rel=1e-9)
    assert T.global_error(t, cand) == pytest.approx(0.07 ** 2, rel=1e-9)
    assert T.global_error(t, T.Trace(np.zeros_like(x), FS)) == 1.0
    r = np.random.default_rng(20240811)
    a = r.standard_normal(256)
    b = a + 0.1 * r.standard_normal(256)
    w3 = T.TimeWindow(128 / FS, 60 / FS)
    assert T.local_error(T.Trace(a, FS), T.Trace(b, FS), w3) == pytest.approx(
        T.local_error(T.Trace(5 * a, FS), T.Trace(5 * b, FS), w3), rel=1e-12)
    with pytest.raises(ValueError):
        z = T.Trace(np.zeros(128), FS)
        T.local_error(z, z, T.TimeWindow(64 / FS, 10 / FS))
    with pytest.raises(ValueError):
        T.global_error(T.Trace(np.ones(10), FS), T.Trace(np.ones(11), FS))


def test_window_bounds_time_mask():  # ref: test_metrics.py:128
    n, t0, c, h = 200, 3e-6, 4.11e-6, 0.293e-6
    lo, hi = window_bounds(n, t0, FS, c, h)
    t = t0 + np.arange(n) / FS
    assert np.array_equal(np.flatnonzero((t >= c - h) & (t <= c + h)), np.arange(lo, hi))


def test_sidelobe_stats():  # ref: test_metrics.py:140-182
    d = np.linspace(10e-3, 30e-3, 101)
    line = np.zeros(101)
    line[50] = 1.0
    assert T.sidelobe_stats(line, d, [20e-3], guard=2)[0] == DB_FLOOR
    line2 = np.full(101, 0.01)
    line2[50] = 1.0
    assert T.sidelobe_stats(line2, d, [20e-3], guard=2, reference=line2)[1] == 0.0
    r = np.random.default_rng(20240811)
    d3 = np.linspace(10e-3, 30e-3, 201)
    ln, rf = np.abs(r.standard_normal(201)) * 0.02, np.abs(r.standard_normal(201)) * 0.02
    ln[100] = rf[100] = 1.0
    a = T.sidelobe_stats(ln, d3, [20e-3], guard=3, reference=rf)
    b = T.sidelobe_stats(10 * ln, d3, [20e-3], guard=3, reference=10 * rf)
    assert a[0] == pytest.approx(b[0], rel=1e-12) and a[1] == pytest.approx(b[1], rel=1e-12)
    d4 = np.linspace(10e-3, 30e-3, 21)
    with pytest.raises(ValueError):
        T.sidelobe_stats(np.ones(21), d4, list(d4), guard=3)
    with pytest.raises(ValueError):
        T.sidelobe_stats(np.ones(21), d4, [50e-3], guard=1)
    hand = np.full(11, 0.1)
    hand[5] = 2.0
    assert T.sidelobe_stats(hand, np.linspace(0, 1, 11), [0.5], guard=1)[0] == pytest.approx(
        20 * np.log10(0.05), rel=1e-9)


def test_metrics_report(tmp_path, probe):  # ref: test_metrics.py:186, :199
    rep = T.MetricsReport(peak_time=1e-5, peak_amplitude=3.2, fwhm_time=2e-7, fwhm_axial=1.5e-4,
                          local_error=0.01, global_error=0.02, mean_sl_db=-30.0, relative_sl_error=0.1)
    p = tmp_path / "m.csv"
    write_reports(p, [rep, rep])
    lines = p.read_text().splitlines()
    assert lines[0] == ",".join(T.MetricsReport.COLUMNS) and len(lines) == 3
    assert float(lines[1].split(",")[1]) == pytest.approx(3.2)
    r2 = T.MetricsReport(peak_time=0.0, peak_amplitude=1.0, fwhm_time=2.1e-7,
                         fwhm_axial=probe.sound_speed * 2.1e-7 / 2.0, local_error=0.0, global_error=0.0)
    assert r2.fwhm_axial == pytest.approx(1.6170e-4, rel=1e-3)


# ------------------------------------------- test_tidas.py (host containers)


def test_time_window():  # ref: test_tidas.py:54, :58
    with pytest.raises(ValueError):
        T.TimeWindow(1e-6, 0.0)
    w = T.TimeWindow(1e-6, 2e-7).recenter(9e-6)
    assert w.center == 9e-6 and w.half_width == 2e-7


def test_theta_matrix_container(tmp_path):  # ref: test_tidas.py:294, :308, :317
    r = np.random.default_rng(20240811)
    vals = r.uniform(0.5, 1.5, (5, 7))
    m = T.ThetaMatrix(np.linspace(10e-3, 30e-3, 5), np.linspace(5e-3, 40e-3, 7), vals)
    p1, p2 = tmp_path / "a.csv", tmp_path / "b.csv"
    m.save_csv(p1)
    loaded = T.ThetaMatrix.load_csv(p1)
    assert np.allclose(loaded.values, vals, rtol=1e-8)
    loaded.save_csv(p2)
    assert p1.read_bytes() == p2.read_bytes()
    m2 = T.ThetaMatrix(np.array([10e-3]), np.array([10e-3, 20e-3, 30e-3]), np.array([[1.0, np.nan, 1.2]]))
    th = m2.interpolate_row(10e-3, np.array([10e-3, 20e-3, 30e-3]))
    assert th[1] == 0.0 and th[0] == 1.0 and th[2] == 1.2
    with pytest.raises(ValueError):
        T.ThetaMatrix(np.array([1.0]), np.array([1.0, 2.0]), np.ones((2, 2)))


# ------------------------------------------- test_simulate.py (host parts)


def test_pulse(probe):  # ref: test_simulate.py:20-70
    cfg = T.ProbeConfig(fractional_bandwidth=0.6)
    p = T.make_pulse(cfg)
    assert p.sigma == pytest.approx(8.9233631e-8, rel=1e-6)
    pulse = T.make_pulse(probe)
    tau = np.linspace(0, 2.0 / probe.center_frequency, 40)
    assert np.allclose(pulse.evaluate(tau), -pulse.evaluate(-tau), atol=1e-12)
    assert abs(np.sum(pulse.samples) / np.max(np.abs(pulse.samples))) < 1e-3
    n = 1 << 12
    spec = np.abs(np.fft.rfft(pulse.samples, n))
    peak = np.fft.rfftfreq(n, d=1.0 / probe.sampling_frequency)[np.argmax(spec)]
    assert abs(peak - probe.center_frequency) <= 2 * probe.sampling_frequency / n
    k = np.argmax(np.abs(pulse.samples))
    assert abs(k / probe.sampling_frequency - pulse.duration / 2) < 1.0 / probe.center_frequency


def test_tx_arrival_times(probe):  # ref: test_simulate.py:74-108
    tx = T.Kossoff(0.6)
    ap = T.tx_aperture(25e-3, tx, probe)
    assert T.tx_arrival_time((0.0, 25e-3), 25e-3, ap, probe) == pytest.approx(25e-3 / probe.sound_speed,
                                                                                rel=1e-12)
    x0 = T.element_position(0, probe)
    t = T.tx_arrival_time((3e-3, 20e-3), 25e-3, np.array([0]), probe)
    assert abs(t - np.hypot(3e-3 - x0, 20e-3) / probe.sound_speed) < 1e-9
    xs, c = T.element_positions(ap, probe), probe.sound_speed
    for z in (10e-3, 18e-3, 32e-3, 41e-3):
        brute = max((np.hypot(x, z) - (np.hypot(x, 25e-3) - 25e-3)) / c for x in xs)
        t = T.tx_arrival_time((0.0, z), 25e-3, ap, probe)
        assert t == pytest.approx(brute, rel=1e-12) and t >= z / c - 1e-9
    d = np.linspace(4e-3, 40e-3, 7)
    assert np.allclose(T.tx_arrival_times(d, 25e-3, ap, probe),
                       [T.tx_arrival_time((0.0, z), 25e-3, ap, probe) for z in d], rtol=0, atol=0)


def test_scatterer_set_validation():  # ref: test_simulate.py:179-190
    for bad in (lambda: T.ScattererSet.on_axis([0.0]), lambda: T.ScattererSet.on_axis([]),
                lambda: T.ScattererSet.on_axis([10e-3], [np.inf])):
        with pytest.raises(ValueError):
            bad()


def test_frame_persistence(tmp_path):  # ref: test_simulate.py:193-225 (host frame; no synthesis)
    r = np.random.default_rng(5)
    fr = T.RfFrame(r.standard_normal((16, 300)), 50e6, 0.0, 25e-3, np.arange(-8, 8))
    T.save_frame(fr, tmp_path / "frame")
    back = T.load_frame(tmp_path / "frame")
    assert back.sampling_frequency == fr.sampling_frequency and back.t0 == fr.t0
    assert back.tx_focus_depth == fr.tx_focus_depth
    assert np.array_equal(back.traces, fr.traces.astype("<f4").astype(float))
    assert back.aperture[0] == fr.aperture[0] and back.aperture[-1] == fr.aperture[-1]
    raw = np.frombuffer((tmp_path / "frame.f32").read_bytes(), dtype="<f4")
    assert np.array_equal(raw[:300], fr.traces[0].astype("<f4"))
    jp, bp = T.save_frame(fr, tmp_path / "frame_2.5mm")
    assert jp.name == "frame_2.5mm.json" and bp.name == "frame_2.5mm.f32"
    assert T.load_frame(tmp_path / "frame_2.5mm").traces.shape == fr.traces.shape
    bp.write_bytes(bp.read_bytes()[:-8])
    with pytest.raises(ValueError):
        T.load_frame(tmp_path / "frame_2.5mm")


def test_vectorised_aperture_half_counts_equal_per_depth(probe):
    """das_value / das_line compute every pixel's aperture at once
    (geometry.aperture_half_counts); it must equal rx_aperture depth by depth."""
    from paper_2507_15464_b200.geometry import aperture_half_count, aperture_half_counts
    z = np.linspace(1e-6, 0.06, 1500)
    for rule in (T.FNumber(1.0), T.FNumber(1.5), T.Kossoff(0.6), T.FixedCount(64), T.FixedCount(7)):
        assert np.array_equal(aperture_half_counts(z, rule, probe),
                              [aperture_half_count(v, rule, probe) for v in z])
    with pytest.raises(TypeError):
        aperture_half_counts(z, object(), probe)
