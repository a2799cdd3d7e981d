"""Pin the CPU oracle against the reference's golden vectors (CPU only).

The vectors in tests/golden were produced by tests/golden/make_golden.py, which
imports the reference package and also regenerates the reference's own figure
fixtures byte-identically.
"""
import csv

import numpy as np
import pytest

from oracle import das as od
from oracle import geom
from oracle import simulate as osim
from oracle import tidas as ot
from tests.conftest import GOLDEN
from tests.setups import REF_PROBE, ref_frame_A

P = REF_PROBE
WL = P["c"] / P["f0"]


@pytest.fixture(scope="module")
def frame_A(ref_vectors):
    traces, tx_xs = ref_frame_A(ref_vectors["A_points"])
    assert traces.shape[1] == int(ref_vectors["A_n_samples"])
    return traces, tx_xs


def _rel_to_max(a, b):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b))) / np.max(np.abs(b)))


def test_delayed_sum_bit_identical(frame_A, ref_vectors):
    traces, _ = frame_A
    got = od.delayed_sum(traces, P["fs"], ref_vectors["A_ds_idx"], ref_vectors["A_ds_delays"])
    assert np.array_equal(got, ref_vectors["A_delayed_sum"])


def test_das_psf_bit_identical(frame_A, ref_vectors):
    traces, _ = frame_A
    half = geom.ref_aperture_half(20e-3, ("fnumber", 1.0), P["n_el"], P["pitch"], WL)
    idx = np.arange(-half, half)
    d = geom.receive_delays(1e-3, 20e-3, (idx + 0.5) * P["pitch"], P["c"])
    assert np.array_equal(od.delayed_sum(traces, P["fs"], idx, d), ref_vectors["A_das_psf"])


def test_envelope_matches_scipy_hilbert(frame_A, ref_vectors):
    traces, _ = frame_A
    env = od.envelope(traces[5 + P["n_el"] // 2])
    assert _rel_to_max(env, ref_vectors["A_envelope_row"]) < 1e-14


def test_das_value_fulltrace_and_gather(frame_A, ref_vectors):
    traces, tx_xs = frame_A
    A = od.analytic_signal(traces)
    ref = ref_vectors["A_das_value"]
    full, gath = [], []
    for x, z in zip(ref_vectors["A_px"], ref_vectors["A_pz"]):
        half = geom.ref_aperture_half(z, ("fnumber", 1.0), P["n_el"], P["pitch"], WL)
        ts = float(geom.focused_expected_arrival(x, z, 25e-3, tx_xs, P["c"]))
        full.append(od.das_value_fulltrace(traces, P["fs"], 0.0, x, z, half, P["pitch"], P["c"], ts))
        gath.append(od.das_image(A[None], P["fs"], 0.0, [x], [z], P["pitch"], P["c"],
                                 np.array([[[ts]]]), ("ref", ("fnumber", 1.0), WL))[0, 0])
    assert _rel_to_max(full, ref) < 1e-13
    assert _rel_to_max(gath, ref) < 1e-13


def test_gather_breaks_without_head_zeros():
    """The B.1 precondition is real: wrap the tail into the head and parity goes."""
    rng = np.random.default_rng(3)
    n_el, N, fs, c, pitch = 16, 512, 50e6, 1540.0, 0.2e-3
    x = rng.standard_normal((n_el, N))
    A = od.analytic_signal(x)
    half = 8
    z, xp = 4e-3, 1e-3
    ts = 2 * z / c + 0.37 / fs
    full = od.das_value_fulltrace(x, fs, 0.0, xp, z, half, pitch, c, ts)
    gat = od.das_image(A[None], fs, 0.0, [xp], [z], pitch, c, np.array([[[ts]]]),
                       ("ref", ("fixed", 16), c / 7e6))[0, 0]
    assert abs(full - gat) / abs(full) > 1e-6


def test_window_bounds_and_windowed_line(frame_A, ref_vectors):
    traces, tx_xs = frame_A
    eps = float(ref_vectors["eps"])
    vals = []
    for z in ref_vectors["A_depths"]:
        half = geom.ref_aperture_half(z, ("fnumber", 1.0), P["n_el"], P["pitch"], WL)
        idx = np.arange(-half, half)
        s = od.delayed_sum(traces, P["fs"], idx, geom.receive_delays(0.0, z, (idx + 0.5) * P["pitch"], P["c"]))
        ts = float(geom.focused_expected_arrival(0.0, z, 25e-3, tx_xs, P["c"]))
        vals.append(ot.windowed_envelope_value(s, P["fs"], 0.0, ts, eps))
    assert _rel_to_max(vals, ref_vectors["A_das_line_windowed"]) < 1e-13


def test_theta_row_and_tidas_line(frame_A, ref_vectors):
    traces, tx_xs = frame_A
    eps = float(ref_vectors["eps"])
    depths = ref_vectors["A_depths"]
    th = ot.theta_row_aligned(25e-3, depths, n_el=P["n_el"], pitch=P["pitch"], fs=P["fs"], c=P["c"],
                              f0=P["f0"], fbw=P["fbw"], tx_rule=("kossoff", 0.6),
                              rx_rule=("fnumber", 1.0), half_width=eps)
    ref_th = ref_vectors["A_theta_row"]
    assert np.array_equal(np.isnan(th), np.isnan(ref_th))
    ok = np.isfinite(ref_th)
    np.testing.assert_allclose(th[ok], ref_th[ok], rtol=1e-12)
    fh = geom.ref_aperture_half(25e-3, ("fnumber", 1.0), P["n_el"], P["pitch"], WL)
    fidx = np.arange(-fh, fh)
    fdel = geom.receive_delays(0.0, 25e-3, (fidx + 0.5) * P["pitch"], P["c"])
    ts = geom.focused_expected_arrival(np.zeros_like(depths), depths, 25e-3, tx_xs, P["c"])
    line = ot.tidas_line(traces, P["fs"], 0.0, fidx, fdel, np.where(ok, th, 0.0), ts, eps)
    assert _rel_to_max(line, ref_vectors["A_tidas_line"]) < 1e-12


def test_estimate_theta_aligned(frame_A, ref_vectors):
    traces, tx_xs = frame_A
    eps = float(ref_vectors["eps"])
    fh = geom.ref_aperture_half(22e-3, ("fnumber", 1.0), P["n_el"], P["pitch"], WL)
    th = geom.ref_aperture_half(25e-3, ("fnumber", 1.0), P["n_el"], P["pitch"], WL)
    fi, ti = np.arange(-fh, fh), np.arange(-th, th)
    center = float(geom.focused_expected_arrival(0.0, 25e-3, 25e-3, tx_xs, P["c"]))
    got = ot.estimate_theta_aligned(traces, P["fs"], 0.0, center, eps,
                                    fi, geom.receive_delays(0.0, 22e-3, (fi + 0.5) * P["pitch"], P["c"]),
                                    ti, geom.receive_delays(0.0, 25e-3, (ti + 0.5) * P["pitch"], P["c"]))
    assert got == pytest.approx(float(ref_vectors["A_theta_aligned"]), rel=1e-12)


def _cfg1_lines():
    n_el, pitch, f0, fs, c, fbw = 64, 0.3e-3, 5e6, 20e6, 1540.0, 0.6
    wl = c / f0
    tx_half = geom.ref_aperture_half(20e-3, ("fixed", 64), n_el, pitch, wl)
    traces, tx_xs = ot.reference_frame(20e-3, 20e-3, n_el=n_el, pitch=pitch, fs=fs, c=c, f0=f0,
                                       fbw=fbw, tx_half=tx_half)
    padded = np.zeros((n_el, 2048))
    padded[:, :traces.shape[1]] = traces
    depths = np.linspace(5e-3, 40e-3, 256)
    ts = geom.focused_expected_arrival(np.zeros_like(depths), depths, 20e-3, tx_xs, c)
    A = od.analytic_signal(padded)
    rule = ("fnumber", 1.5)
    das = np.array([od.das_image(A[None], fs, 0.0, [0.0], [z], pitch, c, np.array([[[t]]]),
                                 ("ref", rule, wl))[0, 0] for z, t in zip(depths, ts)])
    # focal PSF FWHM -> epsilon (experiments.py:158-174; tidas.py:130-147)
    h = geom.ref_aperture_half(20e-3, rule, n_el, pitch, wl)
    idx = np.arange(-h, h)
    psf = od.delayed_sum(traces, fs, idx, geom.receive_delays(0.0, 20e-3, (idx + 0.5) * pitch, c))
    env = od.envelope(psf)
    k = int(np.argmax(env))
    half = env[k] / 2
    i = np.flatnonzero(env[:k] < half)[-1]
    j = k + np.flatnonzero(env[k + 1:] < half)[0]
    width = ((j + (env[j] - half) / (env[j] - env[j + 1])) - (i + (half - env[i]) / (env[i + 1] - env[i]))) / fs
    eps = width / 2
    th = ot.theta_row_aligned(20e-3, depths, n_el=n_el, pitch=pitch, fs=fs, c=c, f0=f0, fbw=fbw,
                              tx_rule=("fixed", 64), rx_rule=rule, half_width=eps)
    th = np.where(np.isfinite(th), th, 0.0)
    fidx = np.arange(-h, h)
    fdel = geom.receive_delays(0.0, 20e-3, (fidx + 0.5) * pitch, c)
    tid = ot.tidas_line(padded, fs, 0.0, fidx, fdel, th, ts, eps)
    return das, tid, eps, th


def test_cfg1_tidas_vs_das_anchor(ref_vectors):
    """Reference-native tiDAS-vs-DAS error at cfg1 geometry: 0.0689579."""
    das, tid, eps, th = _cfg1_lines()
    assert eps == pytest.approx(float(ref_vectors["C1_eps"]), rel=1e-12)
    assert _rel_to_max(das, ref_vectors["C1_das_line"]) < 1e-12
    assert _rel_to_max(tid, ref_vectors["C1_tidas_line"]) < 1e-12
    err = od.rel_l2(tid, das)
    assert err == pytest.approx(float(ref_vectors["C1_rel_l2"]), rel=1e-9)
    assert f"{err:.3g}" == "0.069"


def test_fixture_line_csv():
    """Oracle reproduces pkg/figures/tests/fixtures/lines/five_uniform_25mm.csv."""
    rows = list(csv.reader(open(GOLDEN / "fixtures" / "lines" / "five_uniform_25mm.csv")))[1:]
    depths = np.linspace(0.005, 0.042, 40)  # the fixture's grid (CSV depths are rounded to 9 s.f.)
    np.testing.assert_allclose(depths, [float(r[0]) for r in rows], rtol=1e-8)
    das_ref = np.array([float(r[1]) for r in rows])
    tid_ref = np.array([float(r[2]) for r in rows])
    wl = P["c"] / P["f0"]
    tx_half = geom.ref_aperture_half(25e-3, ("kossoff", 0.6), P["n_el"], P["pitch"], wl)
    tx_xs = (np.arange(-tx_half, tx_half) + 0.5) * P["pitch"]
    zs = np.linspace(10e-3, 40e-3, 5)
    xs_el = geom.element_x(P["n_el"], P["pitch"])
    arr = geom.focused_tx_arrival(np.zeros(5), zs, 25e-3, tx_xs, P["c"])
    dist = np.hypot(0.0 - xs_el[None, :], zs[:, None])
    sigma = osim.pulse_sigma(P["f0"], P["fbw"])
    n = int(np.ceil(((arr[:, None] + dist / P["c"]).max() + 8 * sigma) * P["fs"])) + 1
    traces = osim.synthesize(np.zeros(5), zs, np.ones(5), n_el=P["n_el"], pitch=P["pitch"], fs=P["fs"],
                             c=P["c"], f0=P["f0"], fbw=P["fbw"], n_samples=n,
                             tx=("focused", 25e-3, tx_xs))
    A = od.analytic_signal(traces)
    ts = geom.focused_expected_arrival(np.zeros_like(depths), depths, 25e-3, tx_xs, P["c"])
    das = np.array([od.das_image(A[None], P["fs"], 0.0, [0.0], [z], P["pitch"], P["c"], np.array([[[t]]]),
                                 ("ref", ("fnumber", 1.0), wl))[0, 0] for z, t in zip(depths, ts)])
    np.testing.assert_allclose(das, das_ref, rtol=5e-9, atol=1e-12 * das_ref.max())
    assert np.all(tid_ref[:4] == 0.0)  # windows off support at the shallow end give 0 (tidas.py:524-527)


def test_rowconv_oracle_definition_and_adjoint(rng):
    B, nz, nx, T = 3, 5, 37, 9
    g = rng.standard_normal((B, nz, nx))
    y = rng.standard_normal((B, nz, nx))
    K = rng.standard_normal((nz, T))
    H = (T - 1) // 2
    fwd = ot.rowconv_fwd(g, K)
    for b in range(B):
        for i in range(nz):
            full = np.convolve(g[b, i], K[i][::-1], mode="full")  # correlation with K
            np.testing.assert_allclose(fwd[b, i], full[T - 1 - H: T - 1 - H + nx], rtol=1e-12, atol=1e-12)
    adj = ot.rowconv_adj(y, K)
    assert np.sum(fwd * y) == pytest.approx(np.sum(g * adj), rel=1e-12)


def test_build_row_kernels_theta_identity():
    psf = np.abs(np.random.default_rng(1).standard_normal((10, 7)))
    K, th = ot.build_row_kernels_from_psfs(psf, 1)
    np.testing.assert_allclose(th, 1.0)
    np.testing.assert_allclose(K, psf)
    K4, th4 = ot.build_row_kernels_from_psfs(psf, 4)
    r = ot.neighbourhood_reference_rows(10, 4)
    assert list(r) == [2, 2, 2, 2, 6, 6, 6, 6, 9, 9]
    assert th4[2] == pytest.approx(1.0) and th4[6] == pytest.approx(1.0)


# ------------------------------------------------ FFT theta estimator (§8(f)1)

from oracle import theta as oth  # noqa: E402


def read_matrix_csv(name):
    """Depth-indexed matrix written by save_matrix_csv (tidas.py:105-117)."""
    rows = list(csv.reader(open(GOLDEN / "fixtures" / name)))
    cols = np.array([float(v) for v in rows[0][1:]])
    refs = np.array([float(r[0]) for r in rows[1:]])
    vals = np.array([[float(v) for v in r[1:]] for r in rows[1:]])
    return refs, cols, vals


def assert_matches_9g(ours, csv_vals):
    """Equal to the CSV's 9 significant digits, NaN pattern identical."""
    assert np.array_equal(np.isnan(ours), np.isnan(csv_vals))
    ok = ~np.isnan(csv_vals)
    np.testing.assert_allclose(ours[ok], csv_vals[ok], rtol=1e-8, atol=0.0)


def test_oracle_error_sweep_reproduces_fixtures(ref_vectors):
    """theta_matrix / error_local / error_global / error_mask CSVs of
    run_error_sweep (experiments.py:334-361) at the fixture config: 40 depths
    5-42 mm, 7 MHz, Tx focus 25 mm, Kossoff 0.6, F#1, eps from the focal FWHM."""
    refs, cols, th_csv = read_matrix_csv("theta_matrix.csv")
    _, _, loc_csv = read_matrix_csv("error_local.csv")
    _, _, glo_csv = read_matrix_csv("error_global.csv")
    _, _, mask_csv = read_matrix_csv("error_mask.csv")
    depths = np.linspace(0.005, 0.042, 40)
    np.testing.assert_allclose(cols, depths, rtol=1e-8)
    th, loc, glo = oth.error_sweep(depths, depths, REF_PROBE, tx_focus=25e-3,
                                   half_width=float(ref_vectors["eps"]))
    assert_matches_9g(th, th_csv)
    assert_matches_9g(loc, loc_csv)
    assert_matches_9g(glo, glo_csv)
    mask = np.where(np.isfinite(loc), (loc < 0.05).astype(float), np.nan)
    assert np.array_equal(mask, mask_csv, equal_nan=True)


@pytest.mark.parametrize("form,key", [("beamsum", "F_theta_sweep"), ("per_element", "F_theta_sweep_pe")])
def test_oracle_theta_matrix_sweep_golden(ref_vectors, form, key):
    """theta_matrix_sweep (tidas.py:394-425), both estimator forms, vs the reference."""
    d = ref_vectors["F_depths"]
    ours = oth.theta_matrix_sweep(d, REF_PROBE, tx_focus=25e-3, half_width=float(ref_vectors["eps"]),
                                  form=form)
    ref = ref_vectors[key]
    assert np.array_equal(np.isnan(ours), np.isnan(ref))
    ok = ~np.isnan(ref)
    np.testing.assert_allclose(ours[ok], ref[ok], rtol=1e-11, atol=1e-13)


# ------------------------------------------------------ line metrics (§8(f)3)

from oracle import metrics as om  # noqa: E402


def test_oracle_line_metrics_golden(ref_vectors):
    w = [om.width_at_half_max(r, 50e6) for r in ref_vectors["G_env_rows"]]
    np.testing.assert_allclose(w, ref_vectors["G_half_widths"], rtol=1e-13)
    d = np.linspace(5e-3, 40e-3, 64)
    db, rel = om.sidelobe_stats(ref_vectors["A_tidas_line"], d, [12e-3, 25e-3, 31e-3], 3,
                                reference=ref_vectors["A_das_line"])
    np.testing.assert_allclose([db, rel], ref_vectors["G_sidelobe"], rtol=1e-12)
    with pytest.raises(ValueError):
        om.width_at_half_max(-np.ones(8), 1.0)
    with pytest.raises(ValueError):
        om.width_at_half_max(np.linspace(0, 1, 8), 1.0)  # maximum at the edge


# ---- round 2: the north-star imaging mode pinned to the reference's primitives


def pw_frame_r2(seed):
    """The seeded cfg2 speckle frame of make_golden_r2.py (float32-rounded)."""
    from tests.setups import CFG2
    rng = np.random.default_rng(int(seed))
    sx, sz, a = osim.speckle(rng, CFG2["n_scat"], CFG2["region_x"], CFG2["region_z"])
    rf = osim.synthesize(sx, sz, a, n_el=CFG2["n_el"], pitch=CFG2["pitch"], fs=CFG2["fs"], c=CFG2["c"],
                         f0=CFG2["f0"], fbw=CFG2["fbw"], n_samples=CFG2["n_samples"], tx=("plane", 0.0))
    return rf.astype(np.float32).astype(np.float64)


def test_oracle_plane_wave_hann_gather_vs_reference_primitives():
    """0-degree plane wave + pixel-centred Hann F#1.5 at 256 cfg2 pixels: the
    oracle's analytic gather equals the reference's own composition (Hann weight x
    das._delay_samples summed, metrics.envelope, np.interp at t* = 2z/c;
    tests/golden/make_golden_r2.py)."""
    from tests.setups import CFG2
    g = dict(np.load(GOLDEN / "ref_vectors_r2.npz"))
    rf = pw_frame_r2(g["PW_seed"])
    A = od.analytic_signal(rf)[None]
    xg, zg = np.linspace(*CFG2["x"], CFG2["nx"]), np.linspace(*CFG2["z"], CFG2["nz"])
    got = []
    for iz, ix in zip(g["PW_iz"], g["PW_ix"]):
        x, z = xg[ix], zg[iz]
        ts = geom.plane_wave_expected_arrival(np.array([[x]]), np.array([[z]]), 0.0, CFG2["n_el"],
                                              CFG2["pitch"], CFG2["c"])[None]
        got.append(od.das_image_vectorized(A, CFG2["fs"], 0.0, [x], [z], CFG2["pitch"], CFG2["c"], ts,
                                           CFG2["f_number"])[0, 0])
    assert _rel_to_max(got, g["PW_values"]) < 1e-12
