"""North-star criterion N1: the tiDAS-vs-DAS approximation error, computed on the
GPU and by the float64 oracle on the same seeded inputs, agrees to 3
significant digits — at cfg2 (full grid), cfg4 (K5-built kernels, sampled depth
rows) and cfg5 (int16 frames, sampled frames and rows). cfg1 is covered in
tests/test_gpu_tidas.py and, reference-native, tests/test_gpu_dropin.py.

Error metric: the reference's ``global_error`` (metrics.py:105-112),
||tiDAS - DAS||^2 / ||DAS||^2, float64 on both images. DAS image: K1 + K2
(FP32) against oracle das_image_vectorized (float64). tiDAS image: the row
operator K6 applied to the reflectivity map (rasterised scatterers, or the
cfg4 map itself) with row kernels from K5 (GPU) / oracle lateral_psfs +
build_row_kernels_from_psfs (CPU), neighbourhood 8, 129 taps, dx = the
grid's lateral pitch. Inputs are generated once (the device
simulator, float32 / float64 / int16) and handed to both sides.
"""
import numpy as np
import pytest
import torch

import paper_2507_15464_b200 as tb
from oracle import das as od
from oracle import geom
from oracle import simulate as osim
from oracle import tidas as ot
from tests.setups import CFG2, CFG4, CFG5

pytestmark = pytest.mark.gpu
DEV = "cuda"
NB, TAPS = 8, 129


def probe_kw(cfg):
    return dict(n_el=cfg["n_el"], pitch=cfg["pitch"], fs=cfg["fs"], c=cfg["c"], f0=cfg["f0"], fbw=cfg["fbw"],
                f_number=cfg["f_number"], n_samples=cfg["n_samples"])


def oracle_kernels(z, rows, dx, cfg):
    """Oracle K[rows] (K5 semantics) from the PSFs of the rows and their
    neighbourhood reference rows only."""
    r = ot.neighbourhood_reference_rows(len(z), NB)
    need = np.unique(np.concatenate([rows, r[rows]]))
    psf = ot.lateral_psfs(z[need], TAPS, dx, **probe_kw(cfg))
    at = {int(i): k for k, i in enumerate(need)}
    K = np.zeros((len(rows), TAPS))
    for q, i in enumerate(rows):
        a, b = psf[at[int(r[i])]], psf[at[int(i)]]
        den = float(a @ a)
        K[q] = (float(a @ b) / den if den > 0 else 0.0) * a
    return K


def oracle_das_rows(rf, cfg, x, z, rows):
    A = od.analytic_signal(np.asarray(rf, float))[None]
    zs = z[rows]
    ts = geom.plane_wave_expected_arrival(x[None, :], zs[:, None], 0.0, cfg["n_el"], cfg["pitch"], cfg["c"])[None]
    return od.das_image_vectorized(A, cfg["fs"], 0.0, x, zs, cfg["pitch"], cfg["c"], ts, cfg["f_number"])


def oracle_rowconv_rows(g, K_rows, rows):
    return ot.rowconv_fwd(np.asarray(g, float)[rows][None], K_rows)[0]


def gpu_images(rf_d, g, cfg, x, z, scale=1.0):
    plan = tb.plane_wave_plan(n_el=cfg["n_el"], pitch=cfg["pitch"], fs=cfg["fs"], c=cfg["c"],
                              n_samples=cfg["n_samples"], x=x, z=z, f_number=cfg["f_number"])
    das = tb.das_image(rf_d, plan)
    K, _ = tb.build_row_kernels(z, TAPS, x[1] - x[0], neighbourhood=NB, **probe_kw(cfg))
    tid = tb.tidas_rowconv(torch.as_tensor(np.asarray(g, np.float32)).to(DEV)[None] * scale, K)
    return das.double().cpu().numpy(), tid.double().cpu().numpy(), K


def three_sf(v):
    return f"{v:.3g}"


def n1_cfg2():
    """(err_gpu, err_ref, checks) at cfg2, full 512 x 256 grid."""
    cfg = CFG2
    x, z = np.linspace(*cfg["x"], cfg["nx"]), np.linspace(*cfg["z"], cfg["nz"])
    sx, sz, a = osim.speckle(np.random.default_rng(2025), cfg["n_scat"], cfg["region_x"], cfg["region_z"])
    rf_d = tb.synthesize_batch(sx[None], sz[None], a[None], angles=[0.0], dtype=torch.float32,
                               **{k: cfg[k] for k in ("n_el", "pitch", "fs", "c", "f0", "fbw", "n_samples")})
    g = tb.rasterize(sx, sz, a, x, z)
    das, tid, K = gpu_images(rf_d, g, cfg, x, z)
    err_gpu = od.global_error(das[0], tid[0])
    rows = np.arange(cfg["nz"])
    rf = rf_d[0, 0].double().cpu().numpy()
    das_ref = oracle_das_rows(rf, cfg, x, z, rows)
    Kref = ot.build_row_kernels_from_psfs(ot.lateral_psfs(z, TAPS, x[1] - x[0], **probe_kw(cfg)), NB)[0]
    tid_ref = ot.rowconv_fwd(ot.rasterize(sx, sz, a, x, z)[None], Kref)[0]
    err_ref = od.global_error(das_ref, tid_ref)
    return err_gpu, err_ref, {"das_rel_l2": od.rel_l2(das[0], das_ref),
                              "K_rel_l2": od.rel_l2(K.double().cpu().numpy(), Kref)}


def test_n1_cfg2_full_grid():
    err_gpu, err_ref, chk = n1_cfg2()
    assert chk["das_rel_l2"] < 1e-5 and chk["K_rel_l2"] < 1e-6
    assert three_sf(err_gpu) == three_sf(err_ref), (err_gpu, err_ref)


def n1_cfg4():
    """(err_gpu, err_ref, checks) at cfg4, 16 sampled depth rows of one map."""
    cfg = CFG4
    x, z = np.linspace(*cfg["x"], cfg["nx"]), np.linspace(*cfg["z"], cfg["nz"])
    r = np.random.default_rng(44)
    g = (r.random((cfg["nz"], cfg["nx"])) < cfg["density"]) * r.standard_normal((cfg["nz"], cfg["nx"]))
    iz, ix = np.nonzero(g)
    rf_d = tb.synthesize_batch(x[ix][None], z[iz][None], g[iz, ix][None], angles=[0.0], dtype=torch.float64,
                               **{k: cfg[k] for k in ("n_el", "pitch", "fs", "c", "f0", "fbw", "n_samples")})
    das, tid, K = gpu_images(rf_d, g, cfg, x, z)
    rows = np.linspace(40, cfg["nz"] - 41, 16).astype(int)
    err_gpu = od.global_error(das[0][rows], tid[0][rows])
    das_ref = oracle_das_rows(rf_d[0, 0].cpu().numpy(), cfg, x, z, rows)
    K_rows = oracle_kernels(z, rows, x[1] - x[0], cfg)
    tid_ref = oracle_rowconv_rows(g, K_rows, rows)
    err_ref = od.global_error(das_ref, tid_ref)
    return err_gpu, err_ref, {"das_rel_l2": od.rel_l2(das[0][rows], das_ref),
                              "K_rel_l2": od.rel_l2(K.double().cpu().numpy()[rows], K_rows)}


def test_n1_cfg4_k5_kernels_sampled_rows():
    err_gpu, err_ref, chk = n1_cfg4()
    assert chk["das_rel_l2"] < 1e-5 and chk["K_rel_l2"] < 1e-6
    assert three_sf(err_gpu) == three_sf(err_ref), (err_gpu, err_ref)


def n1_cfg5(frame):
    """(err_gpu, err_ref, checks) at cfg5 frame ``frame``, 24 sampled rows."""
    cfg = CFG5
    x, z = np.linspace(*cfg["x"], cfg["nx"]), np.linspace(*cfg["z"], cfg["nz"])
    sx, sz, a = osim.speckle(np.random.default_rng(5000 + frame), cfg["n_scat"], cfg["x"], cfg["z"])
    f64 = tb.synthesize_batch(sx[None], sz[None], a[None], angles=[0.0], dtype=torch.float64,
                              **{k: cfg[k] for k in ("n_el", "pitch", "fs", "c", "f0", "fbw", "n_samples")})
    std = tb.frame_std(f64)
    q = tb.quantize_int16(f64, cfg["target_std"], std=std)
    scale = cfg["target_std"] / float(std[0])  # the echoes' scale in the int16 frame
    g = tb.rasterize(sx, sz, a, x, z)
    das, tid, K = gpu_images(q, g, cfg, x, z, scale=scale)
    rows = np.linspace(30, cfg["nz"] - 31, 24).astype(int)
    err_gpu = od.global_error(das[0][rows], tid[0][rows])
    das_ref = oracle_das_rows(q[0, 0].cpu().numpy().astype(np.float64), cfg, x, z, rows)
    K_rows = oracle_kernels(z, rows, x[1] - x[0], cfg)
    tid_ref = oracle_rowconv_rows(ot.rasterize(sx, sz, a, x, z) * scale, K_rows, rows)
    err_ref = od.global_error(das_ref, tid_ref)
    return err_gpu, err_ref, {"das_rel_l2": od.rel_l2(das[0][rows], das_ref)}


@pytest.mark.parametrize("frame", [0, 777])
def test_n1_cfg5_int16_sampled_frames(frame):
    err_gpu, err_ref, chk = n1_cfg5(frame)
    assert chk["das_rel_l2"] < 1e-5
    assert three_sf(err_gpu) == three_sf(err_ref), (err_gpu, err_ref)
