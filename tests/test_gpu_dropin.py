"""GPU parity of the drop-in reference API against the reference's golden vectors.

The calls below are the reference's own (pkg/src/tidas/__init__.py surface);
expected values come from tests/golden/ref_vectors.npz (reference outputs) and
the regenerated reference fixture CSVs.
"""
import csv

import numpy as np
import pytest

import paper_2507_15464_b200 as T
from oracle import das as od
from tests.conftest import GOLDEN

pytestmark = pytest.mark.gpu

PROBE = T.ProbeConfig()
RX, TX = T.FNumber(1.0), T.Kossoff(0.6)


def rel_to_max(a, b):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b))) / np.max(np.abs(b)))


@pytest.fixture(scope="module")
def frame(ref_vectors):
    f = T.synthesize_frame(T.ScattererSet.from_points(ref_vectors["A_points"]), 25e-3, PROBE, TX)
    assert f.n_samples == int(ref_vectors["A_n_samples"])
    return f


def test_synthesize_frame_matches_reference_model(frame, ref_vectors):
    from tests.setups import ref_frame_A
    ref, _ = ref_frame_A(ref_vectors["A_points"])
    assert np.max(np.abs(frame.traces - ref)) <= 1e-12 * np.max(np.abs(ref))


def test_delayed_sum_bit_identical(frame, ref_vectors):
    from paper_2507_15464_b200.das import delayed_sum
    s = delayed_sum(frame, ref_vectors["A_ds_idx"], ref_vectors["A_ds_delays"]).samples
    ref = od.delayed_sum(frame.traces, PROBE.sampling_frequency, ref_vectors["A_ds_idx"],
                         ref_vectors["A_ds_delays"])
    assert np.array_equal(s, ref)  # same arithmetic as numpy, same order


def test_das_psf(frame, ref_vectors):
    psf = T.das_psf(frame, (1e-3, 20e-3), PROBE, RX).samples
    assert rel_to_max(psf, ref_vectors["A_das_psf"]) < 1e-12


def test_envelope(frame, ref_vectors):
    env = T.envelope(T.Trace(frame.traces[frame.row(5)], 50e6)).samples
    assert rel_to_max(env, ref_vectors["A_envelope_row"]) < 1e-12


def test_das_value_off_axis(frame, ref_vectors):
    vals = [T.das_value(frame, (x, z), PROBE, RX) for x, z in zip(ref_vectors["A_px"], ref_vectors["A_pz"])]
    assert rel_to_max(vals, ref_vectors["A_das_value"]) < 1e-12


def test_das_line_and_equals_das_value(frame, ref_vectors):
    depths = ref_vectors["A_depths"]
    line = T.das_line(frame, depths, PROBE, RX)
    assert rel_to_max(line, ref_vectors["A_das_line"]) < 1e-12
    vals = np.array([T.das_value(frame, (0.0, z), PROBE, RX) for z in depths[::8]])
    assert np.array_equal(line[::8], vals)  # test_das.py:239-243


def test_das_line_windowed(frame, ref_vectors):
    line = T.das_line(frame, ref_vectors["A_depths"], PROBE, RX,
                      envelope_half_width=float(ref_vectors["eps"]))
    assert rel_to_max(line, ref_vectors["A_das_line_windowed"]) < 1e-12


def test_theta_row_and_tidas_line(frame, ref_vectors):
    from paper_2507_15464_b200.tidas import theta_row_aligned
    eps = float(ref_vectors["eps"])
    depths = ref_vectors["A_depths"]
    th = theta_row_aligned(25e-3, depths, PROBE, TX, RX, window_half_width=eps)
    ref = ref_vectors["A_theta_row"]
    assert np.array_equal(np.isnan(th), np.isnan(ref))
    ok = np.isfinite(ref)
    np.testing.assert_allclose(th[ok], ref[ok], rtol=1e-10)
    fixed = T.rx_delay_profile(25e-3, T.rx_aperture(25e-3, RX, PROBE), PROBE)
    T.reset_delay_counter()
    line = T.tidas_line(frame, fixed, np.where(ok, ref, 0.0), depths, PROBE, window_half_width=eps)
    assert T.delay_counter() == len(fixed)  # single-pass contract (test_tidas.py:377-386)
    assert rel_to_max(line, ref_vectors["A_tidas_line"]) < 1e-12


def test_estimate_theta_aligned(frame, ref_vectors):
    from paper_2507_15464_b200.tidas import estimate_theta_aligned
    fixed22 = T.rx_delay_profile(22e-3, T.rx_aperture(22e-3, RX, PROBE), PROBE)
    true = T.rx_delay_profile(25e-3, T.rx_aperture(25e-3, RX, PROBE), PROBE)
    win = T.TimeWindow(T.expected_arrival_time((0.0, 25e-3), frame, PROBE), float(ref_vectors["eps"]))
    th = estimate_theta_aligned(frame, win, fixed22, true)
    assert th == pytest.approx(float(ref_vectors["A_theta_aligned"]), rel=1e-12)
    assert estimate_theta_aligned(frame, win, true, true) == 1.0


def test_degenerate_tidas_reduces_to_das(frame, ref_vectors):
    """test_tidas.py:365-375: matched profile, theta = 1 -> windowed DAS value."""
    eps = float(ref_vectors["eps"])
    for depth in (21e-3, 25e-3, 31e-3):
        fixed = T.rx_delay_profile(depth, T.rx_aperture(depth, RX, PROBE), PROBE)
        t = T.tidas_line(frame, fixed, [1.0], np.array([depth]), PROBE, window_half_width=eps)
        d = T.das_line(frame, np.array([depth]), PROBE, RX, envelope_half_width=eps)
        assert t[0] == pytest.approx(d[0], rel=1e-12)


def test_cfg1_anchor_0_0689579(ref_vectors):
    """Reference-native tiDAS-vs-DAS error at cfg1 geometry."""
    p1 = T.ProbeConfig(element_count=64, pitch=0.3e-3, center_frequency=5e6, sampling_frequency=20e6,
                       sound_speed=1540.0, fractional_bandwidth=0.6)
    rx1, tx1 = T.FNumber(1.5), T.FixedCount(64)
    f1 = T.synthesize_frame(T.ScattererSet.on_axis([20e-3]), 20e-3, p1, tx1)
    tr = np.zeros((64, 2048))
    tr[:, :f1.n_samples] = f1.traces
    f1p = T.RfFrame(tr, f1.sampling_frequency, 0.0, f1.tx_focus_depth, f1.aperture)
    psf = T.das_psf(f1, (0.0, 20e-3), p1, rx1)
    eps = T.fwhm_window(psf, T.expected_arrival_time((0.0, 20e-3), f1, p1)).half_width
    assert eps == pytest.approx(float(ref_vectors["C1_eps"]), rel=1e-10)
    d1 = np.linspace(5e-3, 40e-3, 256)
    th = T.theta_row_aligned(20e-3, d1, p1, tx1, rx1, window_half_width=eps)
    th = np.where(np.isfinite(th), th, 0.0)
    fixed = T.rx_delay_profile(20e-3, T.rx_aperture(20e-3, rx1, p1), p1)
    das = T.das_line(f1p, d1, p1, rx1)
    tid = T.tidas_line(f1p, fixed, th, d1, p1, window_half_width=eps)
    assert rel_to_max(das, ref_vectors["C1_das_line"]) < 1e-12
    assert rel_to_max(tid, ref_vectors["C1_tidas_line"]) < 1e-10
    err = np.linalg.norm(tid - das) / np.linalg.norm(das)
    assert f"{err:.3g}" == f"{float(ref_vectors['C1_rel_l2']):.3g}" == "0.069"


def test_fixture_line_csv_das_column():
    rows = list(csv.reader(open(GOLDEN / "fixtures" / "lines" / "five_uniform_25mm.csv")))[1:]
    das_ref = np.array([float(r[1]) for r in rows])
    frame = T.synthesize_frame(T.ScattererSet.on_axis(np.linspace(10e-3, 40e-3, 5)), 25e-3, PROBE, TX)
    line = T.das_line(frame, np.linspace(0.005, 0.042, 40), PROBE, RX)
    np.testing.assert_allclose(line, das_ref, rtol=5e-9, atol=1e-12 * das_ref.max())


def test_reference_errors():
    f = T.RfFrame(np.zeros((192, 2048)), 50e6, 0.0, 25e-3, np.arange(-10, 10))
    with pytest.raises(ValueError):
        T.das_line(f, np.array([10e-3, 9e-3]), PROBE, RX)
    with pytest.raises(ValueError):  # |delay| fs >= n (das.py:87-88)
        T.apply_fractional_delay(T.Trace(np.ones(16), 50e6), 17 / 50e6)
    with pytest.raises(ValueError):
        T.tidas_line(f, T.rx_delay_profile(25e-3, np.arange(-2, 2), PROBE), [1.0, 1.0],
                     np.array([25e-3]), PROBE, window_half_width=1e-7)
    with pytest.raises(ValueError):
        T.tidas_psf(f, T.rx_delay_profile(25e-3, np.arange(-2, 2), PROBE), float("nan"))
    assert T.das_value(f, (0.0, 25e-3), PROBE, RX) == 0.0
    short = T.RfFrame(np.zeros((192, 64)), 50e6, 0.0, 25e-3, np.arange(-10, 10))
    with pytest.raises(ValueError):  # 25 mm F#1 shifts reach 93 samples > 64 (das.py:87-88)
        T.das_value(short, (0.0, 25e-3), PROBE, RX)


def test_fractional_delay_linear_and_spectral(rng):
    x = rng.standard_normal(128)
    for method in ("linear", "spectral"):
        assert np.array_equal(T.apply_fractional_delay(T.Trace(x, 50e6), 0.0, method).samples, x)
    n, cycles, fs = 1024, 65, 50e6
    f0 = cycles * fs / n
    t = np.arange(n) / fs
    sig = np.sin(2 * np.pi * f0 * t)
    delay = 1.0 / (4.0 * f0)
    spec = T.apply_fractional_delay(T.Trace(sig, fs), delay, "spectral").samples
    assert np.max(np.abs(spec - np.sin(2 * np.pi * f0 * (t - delay)))) < 1e-10
