"""GPU parity: K1 (analytic RF) and K2 (fused DAS image) against the oracle.

Tolerance (north star): relative L2 <= 1e-5 for the FP32 kernels against the
float64 oracle; float64 kernels against the reference's golden vectors at
1e-12 of the line maximum.
"""
import numpy as np
import pytest
import torch

import paper_2507_15464_b200 as tb
from oracle import das as od
from oracle import geom
from oracle import simulate as osim
from tests.setups import CFG1, CFG2, CFG3, CFG5, grid, plane_t_star, speckle_rf

pytestmark = pytest.mark.gpu
DEV = "cuda"
FP32_TOL = 1e-5


def rel_l2(a, b):
    return od.rel_l2(np.asarray(a), np.asarray(b))


# ------------------------------------------------------------------ K1


@pytest.mark.parametrize("n", [16, 2048, 4096, 8192])
@pytest.mark.parametrize("dtype", [np.float64, np.float32, np.int16])
def test_analytic_pow2(n, dtype, rng):
    x = (rng.standard_normal((6, n)) * (1000 if dtype == np.int16 else 1)).astype(dtype)
    ref = od.analytic_signal(x.astype(np.float64))
    for prec, tol in (("f64", 1e-13), ("f32", 2e-6)):
        if prec == "f64" and n > 8192:
            continue
        got = tb.rf_analytic(torch.as_tensor(x).to(DEV), prec).cpu().numpy()
        assert np.max(np.abs(got - ref)) / np.max(np.abs(ref)) < tol, (prec, n, dtype)


@pytest.mark.parametrize("n", [17, 100, 1000, 2285, 4096 - 3])
def test_analytic_bluestein_any_length(n, rng):
    x = rng.standard_normal((3, n))
    ref = od.analytic_signal(x)
    got = tb.rf_analytic(torch.as_tensor(x).to(DEV), "f64").cpu().numpy()
    assert np.max(np.abs(got - ref)) / np.max(np.abs(ref)) < 1e-12
    got32 = tb.rf_analytic(torch.as_tensor(x).to(DEV), "f32").cpu().numpy()
    assert np.max(np.abs(got32 - ref)) / np.max(np.abs(ref)) < 5e-6


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_analytic_support_scan_sixteen_samples(prec):
    # N = 16 in FP64 runs one thread per CTA (16 samples per thread): both
    # channels' support slots must still be initialised (found by the K1 fuzz test)
    x = np.zeros((4, 16))
    x[0, 3] = 1.0
    x[1, 0:2] = -1.0
    x[3, 15] = 2.0
    sup = torch.full((4, 2), 99, dtype=torch.int32, device=DEV)
    got = tb.rf_analytic(torch.as_tensor(x).to(DEV), prec, support=sup).cpu().numpy()
    assert sup.cpu().tolist() == [[3, 3], [0, 1], [-1, -1], [15, 15]]
    assert np.max(np.abs(got - od.analytic_signal(x))) < (1e-13 if prec == "f64" else 1e-6)


def test_analytic_support_scan():
    x = np.zeros((3, 64))
    x[0, 10:20] = 1.0
    x[1, 63] = -2.0
    sup = torch.empty((3, 2), dtype=torch.int32, device=DEV)
    tb.rf_analytic(torch.as_tensor(x).to(DEV), "f64", support=sup)
    assert sup.cpu().tolist() == [[10, 19], [63, 63], [-1, -1]]


@pytest.mark.parametrize("dtype", [np.float32, np.int16, np.float64])
def test_analytic_4096_fused_odd_rows_and_support(dtype, rng):
    """FP32 N = 4096 runs the three-pass register kernel: odd row count (last CTA has
    one channel), zero rows and head/tail zeros for the support scan."""
    x = (rng.standard_normal((7, 4096)) * (1000 if dtype == np.int16 else 1)).astype(dtype)
    x[2] = 0
    x[3, :700] = 0
    x[3, 3001:] = 0
    x[6, :4095] = 0
    ref = od.analytic_signal(x.astype(np.float64))
    sup = torch.empty((7, 2), dtype=torch.int32, device=DEV)
    got = tb.rf_analytic(torch.as_tensor(x).to(DEV), "f32", support=sup).cpu().numpy()
    assert np.max(np.abs(got - ref)) / np.max(np.abs(ref)) < 2e-6
    s = sup.cpu().numpy()
    assert s[2].tolist() == [-1, -1] and s[3].tolist() == [700, 3000] and s[6].tolist() == [4095, 4095]
    assert s[0].tolist() == [int(np.flatnonzero(x[0])[0]), int(np.flatnonzero(x[0])[-1])]


@pytest.mark.parametrize("n", [2048, 4096, 8192])
@pytest.mark.parametrize("pad, offset", [(0, 0), (1, 0), (0, 1), (4, 4)])
def test_analytic_strided_rows_through_the_abi(n, pad, offset, rng):
    """Row strides / base pointers that are not 16-byte aligned take the
    non-TMA kernels; aligned ones the TMA-staged / register kernels — every
    combination must give the same analytic rows (C ABI, row stride n + pad)."""
    from paper_2507_15464_b200 import _lib
    rows = 5
    buf = torch.as_tensor(rng.standard_normal(rows * (n + pad) + offset).astype(np.float32)).to(DEV)
    x = buf[offset:offset + rows * (n + pad)].view(rows, n + pad)[:, :n]
    ref = od.analytic_signal(x.cpu().numpy().astype(np.float64))
    out = torch.empty((rows, n), dtype=torch.complex64, device=DEV)
    _lib.check(_lib.lib().tidas_rf_analytic(_lib.ptr(x), _lib.DTYPE_CODE[torch.float32], n + pad, 1.0,
                                           _lib.ptr(out), _lib.PREC_F32, rows, n, None,
                                           _lib.stream_handle(None)))
    got = out.cpu().numpy()
    assert np.max(np.abs(got - ref)) / np.max(np.abs(ref)) < 2e-6


@pytest.mark.parametrize("n", [2048, 4096, 8192])
@pytest.mark.parametrize("dtype", [torch.int16, torch.float32, torch.float64])
def test_analytic_three_pass_unaligned_rows_bitwise(n, dtype):
    """Rows that are not 16-byte aligned take plain loads instead of bulk copies
    (analytic_tp_kernel BULK = false): same arithmetic, so the analytic rows, the
    support scan and a ranged store must equal the aligned run bitwise."""
    g = torch.Generator(device=DEV).manual_seed(n)
    rows = 3
    base = torch.randn(rows * n + 1, device=DEV, generator=g) * 500
    base = base.round().to(dtype) if dtype == torch.int16 else base.to(dtype)
    base[1 + n:1 + n + 37] = 0          # head zeros of row 1
    shifted = base[1:].view(rows, n)     # element offset 1: 2 / 4 / 8 bytes past alignment
    aligned = shifted.clone()
    assert shifted.data_ptr() % 16 != 0 and aligned.data_ptr() % 16 == 0
    sup_a = torch.empty((rows, 2), dtype=torch.int32, device=DEV)
    sup_s = torch.empty((rows, 2), dtype=torch.int32, device=DEV)
    a = tb.rf_analytic(aligned, "f32", scale=0.5, support=sup_a)
    s_ = tb.rf_analytic(shifted, "f32", scale=0.5, support=sup_s)
    assert torch.equal(a, s_) and torch.equal(sup_a, sup_s)
    assert int(sup_a[1, 0]) == 37
    lo, hi = n // 7, n // 2 + 5
    out_a = torch.zeros((rows, n), dtype=torch.complex64, device=DEV)
    out_s = torch.zeros((rows, n), dtype=torch.complex64, device=DEV)
    tb.rf_analytic(aligned, "f32", out=out_a, sample_range=(lo, hi))
    tb.rf_analytic(shifted, "f32", out=out_s, sample_range=(lo, hi))
    assert torch.equal(out_a, out_s) and bool((out_a[:, :lo] == 0).all()) and bool((out_a[:, hi + 1:] == 0).all())


@pytest.mark.parametrize("n,channels,dtype", [(2048, 64, torch.float64), (4096, 128, torch.float32),
                                              (8192, 256, torch.int16)])
def test_analytic_full_size_properties(n, channels, dtype):
    """Size-independent properties of K1 on BASELINE-sized batches (cfg1 / cfg2 / cfg5
    channel counts and trace lengths, 16 frames), no oracle needed: the real part is
    the ingested sample exactly; the transform commutes with a circular shift of the
    row (what lets K2 gather instead of shifting full traces); it is
    linear; and for zero-mean rows with no Nyquist content H(H(x)) = -x."""
    rows = 16 * channels
    g = torch.Generator(device=DEV).manual_seed(n + channels)
    x = torch.randn((rows, n), device=DEV, generator=g) * 300
    x = x.round().to(dtype) if dtype == torch.int16 else x.to(dtype)
    a = tb.rf_analytic(x, "f32")
    assert a.shape == (rows, n) and a.dtype == torch.complex64
    assert torch.equal(a.real, x.to(torch.float32))
    peak = float(a.abs().max())
    shift = n // 3 + 1
    a_s = tb.rf_analytic(torch.roll(x, shift, dims=1).contiguous(), "f32")
    assert float((a_s - torch.roll(a, shift, dims=1)).abs().max()) / peak < 2e-6
    if dtype != torch.int16:  # linearity on the float ingests (an int16 sum could clip)
        y = (torch.randn((rows, n), device=DEV, generator=g) * 300).to(dtype)
        lin = tb.rf_analytic((2 * x - y).contiguous(), "f32")
        assert float((lin - (2 * a - tb.rf_analytic(y, "f32"))).abs().max()) / peak < 4e-6
    # H(H(x)) = -x once DC and Nyquist are removed (the one-sided mask zeroes both in H)
    xf = x.to(torch.float32)
    alt = torch.ones(n, device=DEV)
    alt[1::2] = -1
    xf = xf - xf.mean(dim=1, keepdim=True)
    xf = xf - (xf * alt).mean(dim=1, keepdim=True) * alt
    h = tb.rf_analytic(xf.contiguous(), "f32").imag.contiguous()
    hh = tb.rf_analytic(h, "f32").imag
    assert float((hh + xf).abs().max()) / float(xf.abs().max()) < 4e-6


@pytest.mark.parametrize("n", [2048, 4096, 8192])
@pytest.mark.parametrize("rows", [1, 2, 3])
def test_analytic_register_fft_scale_and_row_counts(n, rows, rng):
    """The three-pass register kernels (N = 2048 / 4096 / 8192) with one, two and
    three rows (a lone last channel) and a non-unit ingest scale on int16."""
    x = (rng.standard_normal((rows, n)) * 1000).astype(np.int16)
    scale = 1e-3
    ref = od.analytic_signal(x.astype(np.float64) * scale)
    sup = torch.empty((rows, 2), dtype=torch.int32, device=DEV)
    got = tb.rf_analytic(torch.as_tensor(x).to(DEV), "f32", scale=scale, support=sup).cpu().numpy()
    assert np.max(np.abs(got - ref)) / np.max(np.abs(ref)) < 2e-6
    nz = [np.flatnonzero(x[r]) for r in range(rows)]
    assert sup.cpu().tolist() == [[int(z[0]), int(z[-1])] for z in nz]


def test_analytic_rejects_short_rows():
    with pytest.raises(ValueError):
        tb.rf_analytic(torch.zeros((2, 3), dtype=torch.float64, device=DEV))


# ------------------------------------------------------------------ K2


def _plane_case(cfg, rf, nz, nx, angles=(0.0,), out="envelope", prec="f32", rf_dtype=torch.float32):
    x, z = grid(cfg, nz, nx)
    plan = tb.plane_wave_plan(n_el=cfg["n_el"], pitch=cfg["pitch"], fs=cfg["fs"], c=cfg["c"],
                              n_samples=rf.shape[-1], x=x, z=z, angles=angles,
                              f_number=cfg["f_number"], out=out, prec=prec)
    img = tb.das_image(torch.as_tensor(rf).to(DEV, rf_dtype), plan).cpu().numpy()
    A = np.stack([od.analytic_signal(np.asarray(rf[f], float)) for f in range(rf.shape[0])])
    ts = plane_t_star(cfg, x, z, angles)
    ref = np.stack([od.das_image_vectorized(A[f], cfg["fs"], 0.0, x, z, cfg["pitch"], cfg["c"], ts,
                                            cfg["f_number"], out=out) for f in range(rf.shape[0])])
    return img, ref, plan


def test_cfg1_psf_image_fp32_f64_input():
    cfg = CFG1
    rf = osim.synthesize([0.0], [20e-3], [1.0], n_el=cfg["n_el"], pitch=cfg["pitch"], fs=cfg["fs"],
                         c=cfg["c"], f0=cfg["f0"], fbw=cfg["fbw"], n_samples=cfg["n_samples"],
                         tx=("plane", 0.0))[None, None]
    img, ref, _ = _plane_case(cfg, rf, cfg["nz"], cfg["nx"], rf_dtype=torch.float64)
    assert rel_l2(img[0], ref[0]) <= FP32_TOL
    # the peak sits at the scatterer
    iz, ix = np.unravel_index(np.argmax(img[0]), img[0].shape)
    x, z = grid(cfg)
    assert abs(z[iz] - 20e-3) < 0.3e-3 and abs(x[ix]) < 0.3e-3


def test_cfg1_fp64_instantiation_tight():
    cfg = CFG1
    rf = osim.synthesize([1e-3], [18e-3], [1.0], n_el=cfg["n_el"], pitch=cfg["pitch"], fs=cfg["fs"],
                         c=cfg["c"], f0=cfg["f0"], fbw=cfg["fbw"], n_samples=cfg["n_samples"],
                         tx=("plane", 0.0))[None, None]
    img, ref, _ = _plane_case(cfg, rf, 64, 32, prec="f64", rf_dtype=torch.float64)
    assert rel_l2(img, ref) < 1e-11


def test_cfg2_speckle_full_grid():
    cfg = CFG2
    rf, _ = speckle_rf(cfg, seed=2)
    img, ref, _ = _plane_case(cfg, rf[None].astype(np.float32), cfg["nz"], cfg["nx"])
    assert rel_l2(img, ref) <= FP32_TOL


def test_cfg3_coherent_compounding_reduced():
    cfg = CFG3
    ang = cfg["angles"]
    frames = [speckle_rf(cfg, seed=30 + f, n_scat=300, angles=ang)[0] for f in range(2)]
    rf = np.stack(frames).astype(np.float32)
    for out in ("coherent", "envelope"):
        img, ref, _ = _plane_case(cfg, rf, 96, 48, angles=ang, out=out)
        assert rel_l2(img, ref) <= FP32_TOL, out


def test_cfg3_angle_shards_sum_to_the_compounded_image():
    """Angle sharding (parallel.compound_angle_shards): out="iq" plans over
    disjoint angle subsets, summed, give the coherent image of all 11 angles
    (oracle <= 1e-5; against the one-plan image only the FP32 add order differs)."""
    from paper_2507_15464_b200 import parallel
    cfg = CFG3
    ang = list(cfg["angles"])
    frames = [speckle_rf(cfg, seed=40 + f, n_scat=300, angles=ang)[0] for f in range(2)]
    rf = np.stack(frames).astype(np.float32)
    nz, nx = 96, 48
    img, ref, _ = _plane_case(cfg, rf, nz, nx, angles=ang, out="coherent")
    x, z = grid(cfg, nz, nx)
    rf_dev = torch.as_tensor(rf, device=DEV)
    total = None
    for world in (2, 3):
        total = None
        for rank in range(world):
            a0, a1 = parallel.shard_range(len(ang), rank, world)
            plan = tb.plane_wave_plan(n_el=cfg["n_el"], pitch=cfg["pitch"], fs=cfg["fs"], c=cfg["c"],
                                      n_samples=cfg["n_samples"], x=x, z=z, angles=ang[a0:a1],
                                      f_number=cfg["f_number"], out="iq")
            iq = tb.das_image(rf_dev[:, a0:a1].contiguous(), plan)
            total = iq if total is None else total + iq
        got = parallel.compound_angle_shards(total).cpu().numpy()   # one process: the magnitude
        assert rel_l2(got, ref) <= FP32_TOL
        assert rel_l2(got, img) <= 2e-6


def test_cfg5_int16_ingest_reduced():
    cfg = CFG5
    rng = np.random.default_rng(5)
    sx, sz, a = osim.speckle(rng, 400, cfg["x"], (8e-3, 55e-3))
    rf = osim.synthesize(sx, sz, a, n_el=cfg["n_el"], pitch=cfg["pitch"], fs=cfg["fs"], c=cfg["c"],
                         f0=cfg["f0"], fbw=cfg["fbw"], n_samples=cfg["n_samples"], tx=("plane", 0.0))
    q = osim.quantize_int16(rf, cfg["target_std"])[None, None]
    img, ref, _ = _plane_case(cfg, q, 64, 64, rf_dtype=torch.int16)
    assert rel_l2(img, ref) <= FP32_TOL


def _subgrid_parity(cfg, rf_host, rf_dev, angles, out, n_rows=24, n_cols=16, seed=0):
    """Full-size GPU image vs the oracle on a seeded row x column sub-grid."""
    x, z = grid(cfg)
    plan = tb.plane_wave_plan(n_el=cfg["n_el"], pitch=cfg["pitch"], fs=cfg["fs"], c=cfg["c"],
                              n_samples=cfg["n_samples"], x=x, z=z, angles=angles,
                              f_number=cfg["f_number"], out=out)
    img = tb.das_image(rf_dev, plan).cpu().numpy()
    assert img.shape == (rf_dev.shape[0], cfg["nz"], cfg["nx"])
    rng = np.random.default_rng(seed)
    ri = np.sort(rng.choice(cfg["nz"], n_rows, replace=False))
    ci = np.sort(rng.choice(cfg["nx"], n_cols, replace=False))
    ts = plane_t_star(cfg, x[ci], z[ri], angles)
    for f in range(rf_dev.shape[0]):
        A = od.analytic_signal(np.asarray(rf_host[f], float))
        ref = od.das_image_vectorized(A, cfg["fs"], 0.0, x[ci], z[ri], cfg["pitch"], cfg["c"], ts,
                                      cfg["f_number"], out=out)
        assert rel_l2(img[f][np.ix_(ri, ci)], ref) <= FP32_TOL


def test_cfg3_full_size_frames_sampled_pixels():
    """cfg3 at its full size: 11 steered plane waves x 128 ch x 4096 f32, 1024 x 512
    image, 2000 speckle scatterers + 5 bright targets, coherent compounding."""
    cfg = CFG3
    ang = list(cfg["angles"])
    rng = np.random.default_rng(33)
    F = 2
    sx = rng.uniform(*cfg["region_x"], (F, cfg["n_scat"] + 5))
    sz = rng.uniform(*cfg["region_z"], (F, cfg["n_scat"] + 5))
    a = rng.standard_normal((F, cfg["n_scat"] + 5))
    a[:, cfg["n_scat"]:] = 20.0
    rf = tb.synthesize_batch(sx, sz, a, angles=ang, n_el=cfg["n_el"], pitch=cfg["pitch"], fs=cfg["fs"],
                             c=cfg["c"], f0=cfg["f0"], fbw=cfg["fbw"], n_samples=cfg["n_samples"])
    _subgrid_parity(cfg, rf.cpu().numpy(), rf, ang, "coherent")


def test_cfg5_full_size_int16_frames_sampled_pixels():
    """cfg5 at its full size: 192 ch x 8192 int16 (std 1000, rounded, clipped),
    1024 x 1024 image, 4000 speckle scatterers."""
    cfg = CFG5
    rng = np.random.default_rng(55)
    F = 2
    sx = rng.uniform(*cfg["x"], (F, cfg["n_scat"]))
    sz = rng.uniform(8e-3, 58e-3, (F, cfg["n_scat"]))
    a = rng.standard_normal((F, cfg["n_scat"]))
    rf = tb.synthesize_batch(sx, sz, a, angles=[0.0], n_el=cfg["n_el"], pitch=cfg["pitch"], fs=cfg["fs"],
                             c=cfg["c"], f0=cfg["f0"], fbw=cfg["fbw"], n_samples=cfg["n_samples"],
                             dtype=torch.float64).cpu().numpy()
    q = np.stack([osim.quantize_int16(rf[f, 0], cfg["target_std"])[None] for f in range(F)])
    assert q.dtype == np.int16 and q.shape == (F, 1, 192, 8192)
    _subgrid_parity(cfg, q, torch.as_tensor(q).to(DEV), [0.0], "envelope")


@pytest.mark.parametrize("cfg,frames,dtype", [(CFG2, 16, torch.float32), (CFG3, 2, torch.float32),
                                              (CFG5, 4, torch.int16)], ids=["cfg2", "cfg3", "cfg5"])
def test_das_full_size_properties(cfg, frames, dtype):
    """Size-independent properties of K1 + K2 at the full BASELINE grids and trace
    lengths (no oracle needed): the IQ image is linear in the RF; frames are
    independent (a permuted batch gives the permuted images bitwise); coherent =
    |IQ|; the envelope image is finite, non-negative, exactly homogeneous under a
    power-of-two gain and, for one transmit, never below |IQ| (np.interp of two
    magnitudes against the magnitude of the interpolated sum)."""
    ang = cfg.get("angles", (0.0,))
    x, z = grid(cfg)
    kw = dict(n_el=cfg["n_el"], pitch=cfg["pitch"], fs=cfg["fs"], c=cfg["c"], n_samples=cfg["n_samples"],
              x=x, z=z, angles=ang, f_number=cfg["f_number"])
    g = torch.Generator(device=DEV).manual_seed(len(ang) * 1000 + frames)
    shape = (frames, len(ang), cfg["n_el"], cfg["n_samples"])
    a = (torch.randn(shape, device=DEV, generator=g) * 200).round()
    b = (torch.randn(shape, device=DEV, generator=g) * 200).round()
    for t in (a, b):  # head / tail zeros, as an acquisition has them
        t[..., :64] = 0
        t[..., -64:] = 0
    iq = tb.plane_wave_plan(out="iq", **kw)
    ia, ib = tb.das_image(a.to(dtype), iq), tb.das_image(b.to(dtype), iq)
    iab = tb.das_image((a - b).to(dtype), iq)   # |a - b| stays far inside int16
    peak = float(ia.abs().max())
    assert peak > 0 and float((iab - (ia - ib)).abs().max()) / peak < 2e-5
    perm = torch.randperm(frames, device=DEV, generator=g)
    assert torch.equal(tb.das_image(a[perm].to(dtype).contiguous(), iq), ia[perm])
    coh = tb.das_image(a.to(dtype), tb.plane_wave_plan(out="coherent", **kw))
    assert float((coh - ia.abs()).abs().max()) / peak < 2e-6
    env_plan = tb.plane_wave_plan(out="envelope", **kw)
    env = tb.das_image(a.to(dtype), env_plan)
    assert bool((env >= 0).all()) and bool(torch.isfinite(env).all())
    assert torch.equal(tb.das_image((4 * a).to(dtype), env_plan), 4 * env)   # exact: power-of-two gain
    if len(ang) == 1:  # one transmit: np.interp of two magnitudes >= the magnitude of the interpolated IQ
        assert bool((env >= ia.abs() * (1 - 1e-5) - 1e-6 * peak).all())


def test_iq_output_and_ragged_grid():
    cfg = CFG2
    rf, _ = speckle_rf(cfg, seed=7, n_scat=200)
    img, ref, _ = _plane_case(cfg, rf[None].astype(np.float32), 37, 53, out="iq")
    assert img.dtype == np.complex64
    assert rel_l2(img, ref) <= FP32_TOL


def test_frame_batching_is_bitwise_per_frame():
    """Frames share the time-of-flight work in a CTA; each frame's image is the
    one it gets alone (worker-count invariance, test_experiments.py:124-131)."""
    cfg = CFG2
    rfs = np.stack([speckle_rf(cfg, seed=40 + f, n_scat=150)[0] for f in range(5)]).astype(np.float32)
    x, z = grid(cfg, 64, 32)
    plan = tb.plane_wave_plan(n_el=cfg["n_el"], pitch=cfg["pitch"], fs=cfg["fs"], c=cfg["c"],
                              n_samples=cfg["n_samples"], x=x, z=z, f_number=cfg["f_number"])
    batch = tb.das_image(torch.as_tensor(rfs).to(DEV), plan).cpu().numpy()
    for f in range(5):
        alone = tb.das_image(torch.as_tensor(rfs[f:f + 1]).to(DEV), plan).cpu().numpy()[0]
        assert np.array_equal(batch[f], alone)


def test_host_pipeline_matches_device_path():
    """HostPipeline (pinned host in/out, 3 streams, double-buffered chunks) is
    bit-identical to das_image on device tensors, across ragged last chunks and
    back-to-back calls that reuse its buffers."""
    cfg = CFG2
    rfs = np.stack([speckle_rf(cfg, seed=60 + f, n_scat=150)[0] for f in range(7)]).astype(np.float32)
    x, z = grid(cfg, 64, 48)
    plan = tb.plane_wave_plan(n_el=cfg["n_el"], pitch=cfg["pitch"], fs=cfg["fs"], c=cfg["c"],
                              n_samples=cfg["n_samples"], x=x, z=z, f_number=cfg["f_number"])
    ref = tb.das_image(torch.as_tensor(rfs).to(DEV), plan).cpu()
    pipe = tb.HostPipeline(plan, chunk=3)
    host_rf = torch.as_tensor(rfs).pin_memory()  # [F][A=1][E][N]
    outs = [torch.empty((7, 64, 48), dtype=torch.float32).pin_memory() for _ in range(3)]
    for o in outs:
        pipe.run(host_rf, o)
    pipe.synchronize()
    for o in outs:
        assert torch.equal(o, ref)
    with pytest.raises(ValueError):
        pipe.run(host_rf.to(DEV), outs[0])
    with pytest.raises(ValueError):
        pipe.run(host_rf.double(), outs[0])


def test_zero_rf_and_out_of_support_pixels():
    cfg = CFG1
    x, z = grid(cfg, 40, 8)
    z = np.concatenate([z, [200e-3]])  # t* beyond the record -> 0 (np.interp right=0)
    plan = tb.plane_wave_plan(n_el=cfg["n_el"], pitch=cfg["pitch"], fs=cfg["fs"], c=cfg["c"],
                              n_samples=cfg["n_samples"], x=x, z=z, f_number=cfg["f_number"])
    zero = torch.zeros((2, 1, cfg["n_el"], cfg["n_samples"]), device=DEV)
    assert not tb.das_image(zero, plan).any()
    rf = osim.synthesize([0.0], [20e-3], [1.0], n_el=cfg["n_el"], pitch=cfg["pitch"], fs=cfg["fs"],
                         c=cfg["c"], f0=cfg["f0"], fbw=cfg["fbw"], n_samples=cfg["n_samples"],
                         tx=("plane", 0.0))
    img = tb.das_image(torch.as_tensor(rf[None, None]).to(DEV), plan).cpu().numpy()
    assert np.all(img[0, -1] == 0.0)
    assert tb.das_image(torch.zeros((0, 1, cfg["n_el"], cfg["n_samples"]), device=DEV), plan).shape[0] == 0


def test_plan_validation():
    cfg = CFG1
    x, z = grid(cfg, 8, 8)
    plan = tb.plane_wave_plan(n_el=cfg["n_el"], pitch=cfg["pitch"], fs=cfg["fs"], c=cfg["c"],
                              n_samples=cfg["n_samples"], x=x, z=z, f_number=cfg["f_number"])
    with pytest.raises(ValueError):
        tb.das_from_analytic(torch.zeros((1, 1, 4, 16), dtype=torch.complex64, device=DEV), plan)


def test_file_ingest_to_images_through_host_pipeline(tmp_path):
    """save_frame blobs -> read_frames_pinned -> HostPipeline == das_image."""
    cfg = CFG2
    bases = []
    rfs = []
    for f in range(3):
        rf, _ = speckle_rf(cfg, seed=80 + f, n_scat=120)
        fr = tb.RfFrame(rf[0], cfg["fs"], 0.0, 0.0, np.arange(-4, 4))
        tb.save_frame(fr, tmp_path / f"frame{f}")
        bases.append(tmp_path / f"frame{f}")
        rfs.append(rf.astype(np.float32))
    host, hdr = tb.read_frames_pinned(bases)
    assert host.is_pinned() and hdr[0]["sampling_frequency"] == cfg["fs"]
    x, z = grid(cfg, 48, 32)
    plan = tb.plane_wave_plan(n_el=cfg["n_el"], pitch=cfg["pitch"], fs=cfg["fs"], c=cfg["c"],
                              n_samples=cfg["n_samples"], x=x, z=z, f_number=cfg["f_number"])
    out = torch.empty((3, 48, 32), dtype=torch.float32).pin_memory()
    pipe = tb.HostPipeline(plan, chunk=2)
    pipe.run(host, out)
    pipe.synchronize()
    ref = tb.das_image(torch.as_tensor(np.stack(rfs)).to(DEV), plan).cpu()
    assert torch.equal(out, ref)


# ------------------------------------------- plan window sizing (TMA staging box)


TILE_Z, TILE_X, NARROW = 16, 16, 134  # K2's FP32 tile and narrow-box capacity (das.cu)


def _tile_windows_numpy(cfg, x, z, angles=(0.0,)):
    """Restatement of K2's per-tile sample window (das.cu pixel_aperture /
    pixel_arrival) over its 16 x 16-pixel tiles: max over tiles and transmits."""
    half = cfg["n_el"] // 2
    X, Z = np.meshgrid(x, z)
    wmax = 0
    for ang in angles:
        ts = (X * np.sin(ang) + Z * np.cos(ang) + 0.5 * (cfg["n_el"] - 1) * cfg["pitch"] * abs(np.sin(ang))) \
            / cfg["c"] + Z / cfg["c"]
        pos = ts * cfg["fs"]
        k0 = np.floor(pos).astype(np.int64)
        a = Z / (2 * cfg["f_number"])
        n_lo = np.maximum(np.floor((X - a) / cfg["pitch"] - 0.5).astype(int), -half)
        n_hi = np.minimum(np.ceil((X + a) / cfg["pitch"] - 0.5).astype(int), half - 1)
        dxm = np.minimum(a, np.maximum(np.abs((n_lo + 0.5) * cfg["pitch"] - X), np.abs((n_hi + 0.5) * cfg["pitch"] - X)))
        m_min = np.floor((Z - np.hypot(dxm, Z)) / cfg["c"] * cfg["fs"]).astype(np.int64) - 1
        act = (pos >= 0) & (pos <= cfg["n_samples"] - 1) & (n_lo <= n_hi)
        for i in range(0, Z.shape[0], TILE_Z):
            for j in range(0, Z.shape[1], TILE_X):
                sl = (slice(i, i + TILE_Z), slice(j, j + TILE_X))
                m = act[sl]
                if m.any():
                    lo = (k0[sl][m] - 1).min()
                    hi = (k0[sl] - m_min[sl])[m].max() + 1
                    wmax = max(wmax, int(hi - lo + 1))
    return wmax


def test_plan_window_matches_restatement_and_boxes_are_bitwise_equal():
    """tidas_das_window == the numpy restatement of K2's tile windows (cfg2 grid:
    129 samples, fits the 136-sample box); images from the narrow and the wide
    (256) staging box are bitwise identical and match the oracle."""
    cfg = CFG2
    rf, _ = speckle_rf(cfg, seed=11, n_scat=400)
    rf = rf[None].astype(np.float32)
    x, z = grid(cfg)
    img, ref, plan = _plane_case(cfg, rf, cfg["nz"], cfg["nx"])
    assert plan.window() == _tile_windows_numpy(cfg, x, z) == 129
    assert rel_l2(img, ref) <= FP32_TOL
    plan._window = 0  # unknown: the widest box
    wide = tb.das_image(torch.as_tensor(rf).to(DEV), plan).cpu().numpy()
    assert np.array_equal(img, wide)


@pytest.mark.parametrize("nz, forced", [(384, None), (384, 100), (512, 100)])
def test_plan_window_wide_and_underestimated(nz, forced):
    """A grid whose tile windows exceed the narrow box (nz = 384: ~150 samples)
    takes the wide box; an underestimated window (forced) picks the narrow box
    and the wider tiles gather from global memory — exact either way."""
    cfg = CFG2
    rf, _ = speckle_rf(cfg, seed=12, n_scat=300)
    rf = rf[None].astype(np.float32)
    x, z = grid(cfg, nz, 64)
    plan = tb.plane_wave_plan(n_el=cfg["n_el"], pitch=cfg["pitch"], fs=cfg["fs"], c=cfg["c"],
                              n_samples=rf.shape[-1], x=x, z=z, f_number=cfg["f_number"])
    assert plan.window() == _tile_windows_numpy(cfg, x, z)
    if nz == 384:
        assert NARROW < plan.window() <= 254
    if forced is not None:
        plan._window = forced
    img = tb.das_image(torch.as_tensor(rf).to(DEV), plan).cpu().numpy()
    A = od.analytic_signal(np.asarray(rf[0], float))
    ref = od.das_image_vectorized(A, cfg["fs"], 0.0, x, z, cfg["pitch"], cfg["c"],
                                  plane_t_star(cfg, x, z, (0.0,)), cfg["f_number"])
    assert rel_l2(img[0], ref) <= FP32_TOL


def test_plan_window_cfg3_steered_and_cfg5():
    """Steered transmits (cfg3, 11 angles) and the cfg5 grid: the device window
    equals the restatement (and both fit the narrow box)."""
    for cfg, angles in ((CFG3, CFG3["angles"]), (CFG5, (0.0,))):
        x, z = grid(cfg)
        plan = tb.plane_wave_plan(n_el=cfg["n_el"], pitch=cfg["pitch"], fs=cfg["fs"], c=cfg["c"],
                                  n_samples=cfg["n_samples"], x=x, z=z, angles=angles,
                                  f_number=cfg["f_number"], out="coherent" if len(angles) > 1 else "envelope")
        w = plan.window()
        assert w == _tile_windows_numpy(cfg, x, z, angles)
        assert 0 < w <= NARROW
