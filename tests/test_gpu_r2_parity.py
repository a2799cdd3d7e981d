"""GPU parity, round 2: the paths round 1 left unpinned or untested.

* the cfg2 imaging mode (0-degree plane wave, pixel-centred Hann F#1.5) against
  the reference's OWN primitives at 256 pixels (tests/golden/make_golden_r2.py);
* the drop-in's full-trace fallback (das.py:220-225 here) on a frame with no
  leading zeros, against the reference's das_value / das_line;
* tidas_psf crop / support semantics (reference tidas.py:336-351) and
  window_signals (tidas.py:150-168);
* the device int16 quantiser (cfg5 ingest) against the oracle, bit-exact;
* argument validation that guards the kernels' output buffers.
"""
import numpy as np
import pytest
import torch

import paper_2507_15464_b200 as tb
from oracle import das as od
from oracle import simulate as osim
from tests.conftest import GOLDEN
from tests.setups import CFG2
from tests.test_oracle import pw_frame_r2

pytestmark = pytest.mark.gpu
DEV = "cuda"


@pytest.fixture(scope="module")
def g2():
    return dict(np.load(GOLDEN / "ref_vectors_r2.npz"))


def rel_to_max(a, b):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b))) / np.max(np.abs(b)))


# ---------------------------------------------------------------- PW + Hann


@pytest.mark.parametrize("prec,tol", [("f64", 1e-11), ("f32", 1e-5)])
def test_cfg2_plane_wave_hann_vs_reference_primitives(g2, prec, tol):
    """Full cfg2 grid through das_image; the 256 golden pixels must match the
    reference's composition: FP64 to 1e-11 of the max, FP32 to 1e-5 rel L2
    (north-star tolerance)."""
    rf = pw_frame_r2(g2["PW_seed"])
    dt = torch.float64 if prec == "f64" else torch.float32
    rf_d = torch.as_tensor(rf[None, None]).to(DEV, dt)
    x, z = np.linspace(*CFG2["x"], CFG2["nx"]), np.linspace(*CFG2["z"], CFG2["nz"])
    plan = tb.plane_wave_plan(n_el=CFG2["n_el"], pitch=CFG2["pitch"], fs=CFG2["fs"], c=CFG2["c"],
                              n_samples=CFG2["n_samples"], x=x, z=z, f_number=CFG2["f_number"], prec=prec)
    img = tb.das_image(rf_d, plan)[0].double().cpu().numpy()
    got = img[g2["PW_iz"], g2["PW_ix"]]
    if prec == "f64":
        assert rel_to_max(got, g2["PW_values"]) < tol
    else:
        assert od.rel_l2(got, g2["PW_values"]) < tol


# ------------------------------------------------- full-trace fallback path


def test_full_trace_fallback_on_frame_without_head_zeros(g2, monkeypatch):
    from paper_2507_15464_b200 import das as ddas
    p1 = tb.ProbeConfig(element_count=64, pitch=0.3e-3, center_frequency=5e6, sampling_frequency=20e6,
                        sound_speed=1540.0, fractional_bandwidth=0.6)
    frame = tb.synthesize_frame(tb.ScattererSet.from_points(g2["NZ_points"]), 20e-3, p1, tb.FixedCount(64),
                                noise_amplitude=0.02, rng=np.random.default_rng(11))
    assert np.all(frame.traces[:, 0] != 0.0)
    decisions = []
    real = ddas._gather_exact

    def spy(*a, **k):
        r = real(*a, **k)
        decisions.append(r)
        return r

    monkeypatch.setattr(ddas, "_gather_exact", spy)
    rx = tb.FNumber(1.5)
    vals = [tb.das_value(frame, (x, z), p1, rx) for x, z in zip(g2["NZ_px"], g2["NZ_pz"])]
    line = tb.das_line(frame, g2["NZ_depths"], p1, rx)
    assert decisions and not any(decisions), "the analytic gather must be rejected on this frame"
    assert rel_to_max(vals, g2["NZ_das_value"]) < 1e-11
    assert rel_to_max(line, g2["NZ_das_line"]) < 1e-11


# ------------------------------------------------ tidas_psf / window_signals


@pytest.fixture(scope="module")
def windowed(g2):
    probe, rx, tx = tb.ProbeConfig(), tb.FNumber(1.0), tb.Kossoff(0.6)
    frame = tb.synthesize_frame(tb.ScattererSet.on_axis([25e-3]), 25e-3, probe, tx)
    w = tb.TimeWindow(float(g2["CR_center"]), float(g2["CR_half_width"]))
    fixed = tb.rx_delay_profile(20e-3, tb.rx_aperture(25e-3, rx, probe), probe)
    return frame, tb.window_signals(frame, w), fixed


def test_window_signals_matches_reference(g2, windowed):
    frame, wf, _ = windowed
    nz = np.flatnonzero(np.any(wf.traces != 0.0, axis=0))
    assert [int(nz[0]), int(nz[-1]) + 1] == g2["WS_bounds"].tolist()
    assert rel_to_max(wf.traces.sum(axis=1), g2["WS_row_sums"]) < 1e-12
    s0, s1 = g2["WS_bounds"]
    assert np.array_equal(wf.traces[:, s0:s1], frame.traces[:, s0:s1])  # no arithmetic on kept samples
    for w, raises in zip((tb.TimeWindow(-1e-6, 1e-7), tb.TimeWindow(frame.times[-1], 1e-6)), g2["WS_raises"]):
        if raises:
            with pytest.raises(ValueError):
                tb.window_signals(frame, w)


def test_tidas_psf_crop_semantics(g2, windowed):
    _, wf, fixed = windowed
    full = tb.tidas_psf(wf, fixed, 1.3).samples
    crop = tb.tidas_psf(wf, fixed, 1.3, crop=True).samples
    narrow = tb.tidas_psf(wf, fixed, 1.3, crop=True, support=tuple(int(v) for v in g2["CR_support"] + [4, -4]))
    assert rel_to_max(full, g2["CR_full"]) < 1e-12
    assert rel_to_max(crop, g2["CR_crop"]) < 1e-12
    assert rel_to_max(narrow.samples, g2["CR_crop_narrow"]) < 1e-12
    assert np.max(np.abs(narrow.samples - full)) > 1e-3 * np.max(np.abs(full))  # the support is honoured
    assert bool(g2["CR_short_raises"])
    with pytest.raises(ValueError):
        tb.tidas_psf(wf, fixed, 1.3, crop=True, support=(0, 1))
    zero = tb.RfFrame(np.zeros_like(wf.traces), wf.sampling_frequency, 0.0, wf.tx_focus_depth, wf.aperture)
    assert not tb.tidas_psf(zero, fixed, 1.3, crop=True).samples.any()


# --------------------------------------------------------- int16 quantiser


@pytest.mark.parametrize("src", ["f64", "f32"])
def test_quantize_int16_bit_exact_vs_oracle(src):
    frames = np.stack([osim.synthesize(*osim.speckle(np.random.default_rng(s), 300, (-20e-3, 20e-3),
                                                      (5e-3, 45e-3)), n_el=32, pitch=0.3e-3, fs=40e6,
                                        c=1540.0, f0=5e6, fbw=0.6, n_samples=2048, tx=("plane", 0.0))
                       for s in range(3)])
    if src == "f32":
        frames = frames.astype(np.float32)
    d = torch.as_tensor(frames).to(DEV)
    std = tb.frame_std(d).cpu().numpy()
    want_std = np.array([np.std(f.astype(np.float64)) for f in frames])
    assert np.allclose(std, want_std, rtol=1e-12, atol=0)
    q = tb.quantize_int16(d, 1000.0).cpu().numpy()
    want = np.stack([osim.quantize_int16(f.astype(np.float64), 1000.0) for f in frames])
    assert q.dtype == np.int16 and np.array_equal(q, want)
    # clipping at the int16 limits and round-half-even
    x = torch.tensor([[0.5, 1.5, 2.5, -0.5, -1.5, 40000.0, -40000.0, 3.0]], dtype=torch.float64, device=DEV)
    qx = tb.quantize_int16(x, 1.0, std=torch.ones(1, dtype=torch.float64)).cpu().numpy()
    assert qx.tolist() == [[0, 2, 2, 0, -2, 32767, -32768, 3]]


def test_synthesize_batch_int16_and_rejected_dtypes():
    sx, sz, a = osim.speckle(np.random.default_rng(3), 200, (-10e-3, 10e-3), (5e-3, 30e-3))
    kw = dict(angles=[0.0], n_el=32, pitch=0.3e-3, fs=40e6, c=1540.0, f0=5e6, fbw=0.6, n_samples=2048)
    q = tb.synthesize_batch(sx[None], sz[None], a[None], dtype=torch.int16, **kw)
    f32 = tb.synthesize_batch(sx[None], sz[None], a[None], dtype=torch.float32, **kw)
    assert q.dtype == torch.int16 and q.shape == f32.shape
    std = float(np.std(f32.double().cpu().numpy()))
    want = np.clip(np.rint(f32.double().cpu().numpy() * (1000.0 / std)), -32768, 32767)
    # same scale up to the order of the f64 std reduction: at most a few
    # half-integer ties may round differently
    assert np.count_nonzero(q.cpu().numpy() != want) <= 2
    for bad in (torch.float16, torch.bfloat16, torch.int32):
        with pytest.raises(ValueError):
            tb.synthesize_batch(sx[None], sz[None], a[None], dtype=bad, **kw)


# ---------------------------------------------------- argument validation


def test_das_image_rejects_mismatched_buffers():
    x, z = np.linspace(-5e-3, 5e-3, 16), np.linspace(10e-3, 20e-3, 16)
    plan = tb.plane_wave_plan(n_el=32, pitch=0.3e-3, fs=40e6, c=1540.0, n_samples=1024, x=x, z=z)
    rf = torch.zeros((2, 1, 32, 1024), device=DEV)
    with pytest.raises(ValueError):  # more channels than the plan
        tb.das_image(torch.zeros((2, 1, 64, 1024), device=DEV), plan)
    with pytest.raises(ValueError):  # fewer transmits than the plan
        tb.das_image(torch.zeros((2, 2, 32, 1024), device=DEV), plan)
    with pytest.raises(ValueError):  # float64 out for an FP32 plan
        tb.das_image(rf, plan, out=torch.zeros((2, 16, 16), dtype=torch.float64, device=DEV))
    with pytest.raises(ValueError):  # out too small
        tb.das_image(rf, plan, out=torch.zeros((1, 16, 16), device=DEV))
    with pytest.raises(ValueError):
        tb.rf_analytic(rf, "f32", out=torch.zeros((2, 1, 32, 512), dtype=torch.complex64, device=DEV))
    with pytest.raises(ValueError):
        tb.rf_analytic(rf, "f32", support=torch.zeros((3, 2), dtype=torch.int32, device=DEV))
    assert tb.das_image(rf, plan).shape == (2, 16, 16)


# ------------------------------------------- guard bands around new outputs


def test_k5_and_quantiser_write_only_their_outputs():
    """Sentinel-filled guard bands after every output of tidas_build_row_kernels
    and tidas_quantize_i16 stay untouched (odd sizes; compute-sanitizer is not
    available on this pool)."""
    from paper_2507_15464_b200 import _lib
    L = _lib.lib()
    nz, taps, pad = 7, 33, 64
    z = torch.as_tensor(np.linspace(6e-3, 14e-3, nz), dtype=torch.float64, device=DEV)
    psf = torch.full((nz * taps + pad,), 7.0, dtype=torch.float64, device=DEV)
    K = torch.full((nz * taps + pad,), 7.0, dtype=torch.float32, device=DEV)
    th = torch.full((nz + pad,), 7.0, dtype=torch.float64, device=DEV)
    _lib.check(L.tidas_build_row_kernels(_lib.ptr(z), nz, taps, 0.15e-3, 32, 0.3e-3, 40e6, 1540.0, 5e6, 0.6, 1.5,
                                         1024, 3, _lib.ptr(psf), _lib.ptr(K), _lib.ptr(th), _lib.stream_handle()))
    torch.cuda.synchronize()
    for buf, n in ((psf, nz * taps), (K, nz * taps), (th, nz)):
        assert bool((buf[n:] == 7.0).all()) and bool(torch.isfinite(buf[:n]).all())
    F, n = 3, 1001
    x = torch.randn((F, n), dtype=torch.float32, device=DEV) * 50
    out = torch.full((F * n + pad,), 1234, dtype=torch.int16, device=DEV)
    std = tb.frame_std(x)
    _lib.check(L.tidas_quantize_i16(_lib.ptr(x), _lib.F32, F, n, _lib.ptr(std), 1000.0, _lib.ptr(out),
                                    _lib.stream_handle()))
    torch.cuda.synchronize()
    assert bool((out[F * n:] == 1234).all())
    assert np.array_equal(out[:F * n].cpu().numpy().reshape(F, n),
                          np.stack([osim.quantize_int16(r.astype(np.float64), 1000.0) for r in x.cpu().numpy()]))
