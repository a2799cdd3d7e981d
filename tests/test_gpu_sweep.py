"""GPU FFT theta estimator and theta / error sweeps vs the
reference's fixtures (theta_matrix.csv, error_local.csv, error_global.csv,
error_mask.csv), golden theta_matrix_sweep vectors and the oracle."""
import numpy as np
import pytest

import paper_2507_15464_b200 as tb
from oracle import geom
from oracle import theta as oth
from tests.setups import REF_PROBE
from tests.test_oracle import assert_matches_9g, read_matrix_csv

pytestmark = pytest.mark.gpu

PROBE = tb.ProbeConfig()  # the reference defaults: 192 el, 0.2 mm, 7 MHz, 50 MHz


def test_error_sweep_reproduces_reference_fixtures(ref_vectors):
    refs, cols, th_csv = read_matrix_csv("theta_matrix.csv")
    _, _, loc_csv = read_matrix_csv("error_local.csv")
    _, _, glo_csv = read_matrix_csv("error_global.csv")
    _, _, mask_csv = read_matrix_csv("error_mask.csv")
    depths = np.linspace(0.005, 0.042, 40)
    th, loc, glo = tb.error_sweep(depths, PROBE, tb.Kossoff(0.6), tb.FNumber(1.0), tx_focus_depth=25e-3,
                                  window_half_width=float(ref_vectors["eps"]))
    assert_matches_9g(th, th_csv)
    assert_matches_9g(loc, loc_csv)
    assert_matches_9g(glo, glo_csv)
    mask = np.where(np.isfinite(loc), (loc < 0.05).astype(float), np.nan)
    assert np.array_equal(mask, mask_csv, equal_nan=True)


@pytest.mark.parametrize("form,key", [("beamsum", "F_theta_sweep"), ("per_element", "F_theta_sweep_pe")])
def test_theta_matrix_sweep_matches_reference(ref_vectors, form, key):
    d = ref_vectors["F_depths"]
    m = tb.theta_matrix_sweep(d, PROBE, tb.Kossoff(0.6), tb.FNumber(1.0), tx_focus_depth=25e-3,
                              window_half_width=float(ref_vectors["eps"]), form=form)
    ref = ref_vectors[key]
    assert isinstance(m, tb.ThetaMatrix) and m.values.shape == ref.shape
    assert np.array_equal(np.isnan(m.values), np.isnan(ref))
    ok = ~np.isnan(ref)
    np.testing.assert_allclose(m.values[ok], ref[ok], rtol=1e-11, atol=1e-13)


def test_theta_sweep_rectangular_and_batched_columns(ref_vectors):
    # more columns than one device batch, explicit reference depths
    targets = np.linspace(6e-3, 40e-3, 131)
    refs = np.array([10e-3, 25e-3, 33e-3])
    eps = float(ref_vectors["eps"])
    m = tb.theta_matrix_sweep(targets, PROBE, tb.Kossoff(0.6), tb.FNumber(1.0), tx_focus_depth=25e-3,
                              window_half_width=eps, reference_depths=refs)
    pick = [0, 47, 96, 130]
    ref = oth.theta_matrix_sweep(targets[pick], REF_PROBE, refs=refs, tx_focus=25e-3, half_width=eps)
    np.testing.assert_allclose(m.values[:, pick], ref, rtol=1e-11, atol=1e-13)


def _windowed_case(ref_vectors, target=20e-3):
    p = REF_PROBE
    wl = p["c"] / p["f0"]
    tx_half = geom.ref_aperture_half(25e-3, ("kossoff", 0.6), p["n_el"], p["pitch"], wl)
    from oracle.tidas import reference_frame
    traces, tx_xs = reference_frame(target, 25e-3, n_el=p["n_el"], pitch=p["pitch"], fs=p["fs"], c=p["c"],
                                    f0=p["f0"], fbw=p["fbw"], tx_half=tx_half)
    center = float(geom.focused_expected_arrival(0.0, target, 25e-3, tx_xs, p["c"]))
    eps = float(ref_vectors["eps"])
    win = oth.window_signals(traces, p["fs"], 0.0, center, eps)
    bounds = oth.window_bounds(traces.shape[1], 0.0, p["fs"], center, eps)
    return win, bounds


@pytest.mark.parametrize("form", ["beamsum", "per_element"])
@pytest.mark.parametrize("use_support", [False, True])
def test_estimate_theta_dropin_vs_oracle(ref_vectors, form, use_support):
    win, bounds = _windowed_case(ref_vectors)
    fr = tb.RfFrame(win, REF_PROBE["fs"], 0.0, 25e-3, np.arange(-4, 4))
    ap = tb.rx_aperture(20e-3, tb.FNumber(1.0), PROBE)
    true = tb.rx_delay_profile(20e-3, ap, PROBE)
    for rd in (12e-3, 20e-3, 31e-3):
        fixed = tb.rx_delay_profile(rd, ap, PROBE)
        got = tb.estimate_theta(fr, fixed, true, form=form, support=bounds if use_support else None)
        want = oth.estimate_theta(win, REF_PROBE["fs"], ap, fixed.delays, true.delays, form,
                                  search=bounds if use_support else None)
        assert got == pytest.approx(want, rel=1e-11)


def test_estimate_theta_errors(ref_vectors):
    win, _ = _windowed_case(ref_vectors)
    fr = tb.RfFrame(win, REF_PROBE["fs"], 0.0, 25e-3, np.arange(-4, 4))
    ap = tb.rx_aperture(20e-3, tb.FNumber(1.0), PROBE)
    true = tb.rx_delay_profile(20e-3, ap, PROBE)
    other = tb.rx_delay_profile(20e-3, ap[1:-1], PROBE)
    with pytest.raises(ValueError):
        tb.estimate_theta(fr, other, true)
    with pytest.raises(ValueError):
        tb.estimate_theta(fr, true, true, form="nope")
    zero = tb.RfFrame(np.zeros_like(win), REF_PROBE["fs"], 0.0, 25e-3, np.arange(-4, 4))
    with pytest.raises(ZeroDivisionError):
        tb.estimate_theta(zero, true, true)
