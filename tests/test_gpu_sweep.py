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


def test_device_cell_geometry_matches_the_host_restatement(ref_vectors):
    """tidas_sweep_theta_geometry_f64 / tidas_sweep_crop_geometry_f64 against the
    numpy cell geometry (tidas.py:254-265, 336-349): FFT lengths, crops and rows
    exactly, delays to a few ulp (CUDA's hypot against glibc's)."""
    import torch
    from paper_2507_15464_b200 import _lib
    from paper_2507_15464_b200 import sweep as sw
    depths = np.linspace(0.005, 0.042, 40)
    refs = depths[::3]
    cols = sw._Columns(depths, PROBE, tb.Kossoff(0.6), 25e-3, float(ref_vectors["eps"]), True)
    from paper_2507_15464_b200.geometry import aperture_half_counts
    halves = aperture_half_counts(depths, tb.FNumber(1.0), PROBE).astype(np.int64)
    good = sw._good_columns(cols)
    R, A, dev = len(refs), int(2 * halves[good].max()), torch.device("cuda")
    C = len(good) * R
    dfx = torch.empty((C, A), dtype=torch.float64, device=dev)
    dtr = torch.empty((C, A), dtype=torch.float64, device=dev)
    nf = torch.empty(C, dtype=torch.int32, device=dev)
    keep = [sw._i32(good, dev), sw._f64(depths, dev), sw._i32(halves, dev),
            sw._i32(cols.s_hi - cols.s_lo, dev), sw._f64(refs, dev)]
    _lib.check(_lib.lib().tidas_sweep_theta_geometry_f64(
        C, R, *[_lib.ptr(k) for k in keep], PROBE.pitch, PROBE.sound_speed, PROBE.sampling_frequency, A,
        _lib.ptr(dfx), _lib.ptr(dtr), _lib.ptr(nf), _lib.stream_handle()))
    dfx, dtr, nf = dfx.cpu().numpy(), dtr.cpu().numpy(), nf.cpu().numpy()
    c = PROBE.sound_speed
    for j, t in enumerate(good):
        idx = np.arange(-halves[t], halves[t])
        xs = tb.element_positions(idx, PROBE)
        d_fix = (refs[:, None] - np.hypot(xs[None, :], refs[:, None])) / c
        d_true = (depths[t] - np.hypot(xs, depths[t])) / c
        df, dt, nfft = sw._cell_geometry(cols, t, idx, d_fix, d_true)
        n = len(idx)
        sl = slice(j * R, (j + 1) * R)
        assert np.array_equal(nf[sl], nfft)
        np.testing.assert_allclose(dfx[sl, :n], df, rtol=0, atol=1e-9)
        np.testing.assert_allclose(dtr[sl, :n], dt, rtol=0, atol=1e-9)
        assert not dfx[sl, n:].any() and not dtr[sl, n:].any()
    # crop mode: every (good column, reference) cell
    t_sel = np.repeat(np.asarray(good), R)
    r_sel = np.tile(np.arange(R), len(good))
    rows, sh, clo, chi, bad, _ = sw._sweep_profiles(cols, halves, sw._i32(t_sel, dev), sw._i32(r_sel, dev),
                                                    sw._f64(refs, dev), PROBE, A)
    rows, sh, clo, chi = (v.cpu().numpy() for v in (rows, sh, clo, chi))
    assert int(bad.item()) == 0
    fs = PROBE.sampling_frequency
    for i, (t, r) in enumerate(zip(t_sel, r_sel)):
        idx = np.arange(-halves[t], halves[t])
        d = (refs[r] - np.hypot(tb.element_positions(idx, PROBE), refs[r])) / c
        span = int(np.ceil(-d.min() * fs)) + 2
        assert clo[i] == max(int(cols.wlo[t]) - span, 0) and chi[i] == min(int(cols.whi[t]) + 2, int(cols.n_len[t]))
        assert np.array_equal(rows[i, :len(idx)], t * PROBE.element_count + idx + PROBE.element_count // 2)
        assert (rows[i, len(idx):] == cols.zero_row).all() and not sh[i, len(idx):].any()
        np.testing.assert_allclose(sh[i, :len(idx)], d * fs, rtol=0, atol=1e-9)
