"""GPU parity of the tiDAS row operator (K6 / K7) and the kernel builder (K5).

No reference counterpart exists: parity is against the
float64 oracle restatement (oracle/tidas.py), the adjoint identity, and the
DAS kernel the builder is defined through.
"""
import numpy as np
import pytest
import torch

import paper_2507_15464_b200 as tb
from oracle import das as od
from oracle import geom
from oracle import simulate as osim
from oracle import tidas as ot
from tests.setups import CFG1, CFG2, CFG4, grid, plane_t_star

pytestmark = pytest.mark.gpu
DEV = "cuda"


def sparse_maps(rng, B, nz, nx, p=0.02):
    return ((rng.random((B, nz, nx)) < p) * rng.standard_normal((B, nz, nx))).astype(np.float32)


@pytest.mark.parametrize("shape", [(2, 64, 256), (3, 7, 1024), (1, 5, 36), (2, 3, 37), (4, 9, 8)])
@pytest.mark.parametrize("taps", [129, 1, 3, 31])
def test_rowconv_fwd_adj_vs_oracle(shape, taps, rng):
    B, nz, nx = shape
    g = sparse_maps(rng, B, nz, nx, 0.2)
    K = rng.standard_normal((nz, taps)).astype(np.float32)
    Kd = torch.as_tensor(K).to(DEV)
    y = tb.tidas_rowconv(torch.as_tensor(g).to(DEV), Kd).cpu().numpy()
    yref = ot.rowconv_fwd(g, K)
    assert od.rel_l2(y, yref) < 1e-6
    a = tb.tidas_rowconv_adjoint(torch.as_tensor(yref.astype(np.float32)).to(DEV), Kd).cpu().numpy()
    aref = ot.rowconv_adj(yref.astype(np.float32), K)
    assert od.rel_l2(a, aref) < 1e-6


def test_rowconv_cfg4_map_size_and_adjoint_identity(rng):
    cfg = CFG4
    B, nz, nx, T = 2, cfg["nz"], cfg["nx"], cfg["taps"]
    g = sparse_maps(rng, B, nz, nx, cfg["density"])
    yv = rng.standard_normal((B, nz, nx)).astype(np.float32)
    K = rng.standard_normal((nz, T)).astype(np.float32) / 8
    Kd = torch.as_tensor(K).to(DEV)
    gd, yd = torch.as_tensor(g).to(DEV), torch.as_tensor(yv).to(DEV)
    Ag = tb.tidas_rowconv(gd, Kd)
    Aty = tb.tidas_rowconv_adjoint(yd, Kd)
    assert od.rel_l2(Ag[:1].cpu().numpy(), ot.rowconv_fwd(g[:1], K)) < 1e-6
    lhs = torch.sum(Ag.double() * yd.double()).item()
    rhs = torch.sum(gd.double() * Aty.double()).item()
    scale = torch.linalg.norm(Ag.double()).item() * torch.linalg.norm(yd.double()).item()
    assert abs(lhs - rhs) / scale < 1e-6


# tensor-core path (tcgen05 3xTF32, batch >= 32, nx % 32 == 0): ragged map
# blocks (B not a multiple of 64), ragged column blocks (nx not a multiple of
# the 64-output block), short and full-width kernels. Tolerance: 2e-6 relative
# L2 vs the float64 oracle (the split drops the lo*lo term and truncates lo,
# ~2^-21 relative per product).
# Every chunk-count edge of the halo-free chunk schedule (a block reads input
# chunks max(0, j - 2) .. min(n_xb - 1, j + 2)): n_xb = 1, 2, 3, 4, 5, 8, 32.
@pytest.mark.parametrize("shape", [(128, 3, 256), (40, 5, 96), (33, 2, 32), (200, 3, 1024), (257, 2, 64),
                                   (96, 2, 128), (64, 3, 160)])
@pytest.mark.parametrize("taps", [129, 31, 1])
def test_rowconv_tensor_core_path_vs_oracle(shape, taps, rng):
    B, nz, nx = shape
    g = sparse_maps(rng, B, nz, nx, 0.2)
    K = rng.standard_normal((nz, taps)).astype(np.float32)
    Kd, gd = torch.as_tensor(K).to(DEV), torch.as_tensor(g).to(DEV)
    y = tb.tidas_rowconv(gd, Kd, path="tensor").cpu().numpy()
    assert od.rel_l2(y, ot.rowconv_fwd(g, K)) < 2e-6
    a = tb.tidas_rowconv_adjoint(gd, Kd, path="tensor").cpu().numpy()
    assert od.rel_l2(a, ot.rowconv_adj(g, K)) < 2e-6


def test_rowconv_tensor_path_rejects_small_batches(rng):
    g = torch.zeros((8, 2, 64), device=DEV)
    K = torch.zeros((2, 129), device=DEV)
    with pytest.raises(NotImplementedError):
        tb.tidas_rowconv(g, K, path="tensor")
    with pytest.raises(ValueError):
        tb.tidas_rowconv(g, K, out=g)  # in place is rejected


def test_rowconv_tensor_core_matches_cuda_core_path(rng):
    B, nz, nx, T = 96, 16, 512, 129
    g = torch.as_tensor(sparse_maps(rng, B, nz, nx, 0.05)).to(DEV)
    K = torch.as_tensor(rng.standard_normal((nz, T)).astype(np.float32) / 8).to(DEV)
    y_tc, a_tc = tb.tidas_rowconv(g, K, path="tensor"), tb.tidas_rowconv_adjoint(g, K, path="tensor")
    y_s, a_s = tb.tidas_rowconv(g, K, path="simt"), tb.tidas_rowconv_adjoint(g, K, path="simt")
    for u, v in ((y_tc, y_s), (a_tc, a_s)):
        assert (torch.linalg.norm((u - v).double()) / torch.linalg.norm(v.double())).item() < 2e-6


@pytest.mark.parametrize("shape,taps", [((64, 3, 30), 129), ((40, 5, 100), 129), ((64, 2, 256), 131)])
def test_rowconv_shapes_outside_tensor_path_fall_back(shape, taps, rng):
    # nx % 32 != 0 (whole 32-input chunks) and taps > 129 run on the CUDA-core kernels
    B, nz, nx = shape
    g = sparse_maps(rng, B, nz, nx, 0.2)
    K = rng.standard_normal((nz, taps)).astype(np.float32)
    y = tb.tidas_rowconv(torch.as_tensor(g).to(DEV), torch.as_tensor(K).to(DEV)).cpu().numpy()
    assert od.rel_l2(y, ot.rowconv_fwd(g, K)) < 1e-6


def test_rowconv_cfg4_full_batch_tensor_core_adjoint_identity():
    # all 256 cfg4 maps through the tensor path: <A g, y> = <g, A^T y>
    cfg = CFG4
    B, nz, nx, T = 256, cfg["nz"], cfg["nx"], cfg["taps"]
    gen = torch.Generator(device=DEV).manual_seed(3)
    g = (torch.rand((B, nz, nx), device=DEV, generator=gen) < cfg["density"]).float() * \
        torch.randn((B, nz, nx), device=DEV, generator=gen)
    yv = torch.randn((B, nz, nx), device=DEV, generator=gen)
    K = torch.randn((nz, T), device=DEV, generator=gen) / 8
    Ag = tb.tidas_rowconv(g, K)
    lhs = torch.sum(Ag.double() * yv.double()).item()
    del Ag
    Aty = tb.tidas_rowconv_adjoint(yv, K)
    rhs = torch.sum(g.double() * Aty.double()).item()
    scale = torch.linalg.norm(g.double()).item() * torch.linalg.norm(yv.double()).item() * \
        torch.linalg.norm(K.double()).item()
    assert abs(lhs - rhs) / scale < 1e-6
    # one map against the oracle at full size
    g0 = g[:1].cpu().numpy()
    y0 = tb.tidas_rowconv(g, K)[:1].cpu().numpy()
    assert od.rel_l2(y0, ot.rowconv_fwd(g0, K.cpu().numpy())) < 2e-6


def test_rowconv_rejects_bad_taps():
    with pytest.raises(ValueError):
        tb.tidas_rowconv(torch.zeros((1, 2, 8), device=DEV), torch.zeros((2, 4), device=DEV))


def _psf_case(cfg, depths, taps, dx):
    return dict(n_el=cfg["n_el"], pitch=cfg["pitch"], fs=cfg["fs"], c=cfg["c"], f0=cfg["f0"],
                fbw=cfg["fbw"], f_number=cfg["f_number"], n_samples=cfg["n_samples"])


def test_lateral_psfs_and_row_kernels_cfg1():
    cfg = CFG1
    x, z = grid(cfg)
    dx = x[1] - x[0]
    kw = _psf_case(cfg, z, 129, dx)
    sub = z[::16]
    got = tb.lateral_psfs(sub, 129, dx, **kw).cpu().numpy()
    ref = ot.lateral_psfs(sub, 129, dx, **kw)
    # K5 is float64 end to end (exact discrete Hilbert kernel instead of the FFT)
    assert got.dtype == np.float64 and od.rel_l2(got, ref) < 1e-10
    K, th = tb.build_row_kernels(sub, 129, dx, neighbourhood=4, **kw)
    Kref, thref = ot.build_row_kernels_from_psfs(ref, 4)
    assert K.dtype == torch.float32 and od.rel_l2(K.double().cpu().numpy(), Kref) < 1e-7
    np.testing.assert_allclose(th.cpu().numpy(), thref, rtol=1e-9)


def test_cfg1_das_vs_tidas_image_error_matches_oracle():
    """cfg1: DAS image of the (0, 20 mm) scatterer vs the tiDAS row-operator image
    of its rasterised reflectivity; the approximation error agrees with the
    oracle's to 3 significant digits."""
    cfg = CFG1
    x, z = grid(cfg)
    dx = x[1] - x[0]
    kw = _psf_case(cfg, z, 129, dx)
    rf = osim.synthesize([0.0], [20e-3], [1.0], n_el=cfg["n_el"], pitch=cfg["pitch"], fs=cfg["fs"],
                         c=cfg["c"], f0=cfg["f0"], fbw=cfg["fbw"], n_samples=cfg["n_samples"],
                         tx=("plane", 0.0))
    plan = tb.plane_wave_plan(n_el=cfg["n_el"], pitch=cfg["pitch"], fs=cfg["fs"], c=cfg["c"],
                              n_samples=cfg["n_samples"], x=x, z=z, f_number=cfg["f_number"])
    das_gpu = tb.das_image(torch.as_tensor(rf[None, None]).to(DEV), plan)[0]
    K, _ = tb.build_row_kernels(z, 129, dx, neighbourhood=8, **kw)
    g = torch.as_tensor(tb.rasterize([0.0], [20e-3], [1.0], x, z).astype(np.float32)).to(DEV)
    tid_gpu = tb.tidas_rowconv(g, K)
    err_gpu = od.rel_l2(tid_gpu.double().cpu().numpy(), das_gpu.double().cpu().numpy())
    # oracle
    A = od.analytic_signal(rf)[None]
    das_ref = od.das_image_vectorized(A, cfg["fs"], 0.0, x, z, cfg["pitch"], cfg["c"],
                                      plane_t_star(cfg, x, z), cfg["f_number"])
    Kref, _ = ot.build_row_kernels_from_psfs(ot.lateral_psfs(z, 129, dx, **kw), 8)
    tid_ref = ot.rowconv_fwd(ot.rasterize([0.0], [20e-3], [1.0], x, z), Kref)
    err_ref = od.rel_l2(tid_ref, das_ref)
    assert od.rel_l2(das_gpu.cpu().numpy(), das_ref) < 1e-5
    assert od.rel_l2(tid_gpu.double().cpu().numpy(), tid_ref) < 1e-5
    assert f"{err_gpu:.3g}" == f"{err_ref:.3g}"


def test_frame_shard_gather_invariance():
    """Per-frame images do not depend on how frames are split (1 vs 3 shards)."""
    from paper_2507_15464_b200.parallel import shard_range
    cfg = CFG2
    rng = np.random.default_rng(9)
    rfs = np.stack([osim.synthesize(*osim.speckle(rng, 100, cfg["region_x"], cfg["region_z"]),
                                    n_el=cfg["n_el"], pitch=cfg["pitch"], fs=cfg["fs"], c=cfg["c"],
                                    f0=cfg["f0"], fbw=cfg["fbw"], n_samples=cfg["n_samples"],
                                    tx=("plane", 0.0))[None] for _ in range(7)]).astype(np.float32)
    x, z = grid(cfg, 64, 32)
    plan = tb.plane_wave_plan(n_el=cfg["n_el"], pitch=cfg["pitch"], fs=cfg["fs"], c=cfg["c"],
                              n_samples=cfg["n_samples"], x=x, z=z, f_number=cfg["f_number"])
    full = tb.das_image(torch.as_tensor(rfs).to(DEV), plan)
    parts = []
    for r in range(3):
        a, b = shard_range(7, r, 3)
        parts.append(tb.das_image(torch.as_tensor(rfs[a:b]).to(DEV), plan))
    assert torch.equal(full, torch.cat(parts))
