"""Empty and minimal inputs through the public entry points (GPU)."""
import numpy as np
import pytest
import torch

import paper_2507_15464_b200 as tb
from tests.setups import CFG2, grid

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _plan(nz=16, nx=8):
    c = CFG2
    x, z = grid(c, nz, nx)
    return tb.plane_wave_plan(n_el=c["n_el"], pitch=c["pitch"], fs=c["fs"], c=c["c"], n_samples=c["n_samples"],
                              x=x, z=z, f_number=c["f_number"])


def test_das_image_zero_frames():
    plan = _plan()
    rf = torch.zeros((0, 1, CFG2["n_el"], CFG2["n_samples"]), device=DEV)
    img = tb.das_image(rf, plan)
    assert img.shape == (0, 16, 8)


def test_rf_analytic_zero_rows():
    out = tb.rf_analytic(torch.zeros((0, 4096), device=DEV), "f32")
    assert out.shape == (0, 4096)


def test_rowconv_zero_maps_and_single_row():
    K = torch.randn((4, 9), device=DEV)
    y = tb.tidas_rowconv(torch.zeros((0, 4, 32), device=DEV), K)
    assert y.shape == (0, 4, 32)
    g = torch.randn((1, 4, 1), device=DEV)  # one column: only the centre tap touches data
    y = tb.tidas_rowconv(g, K)
    assert torch.allclose(y[0, :, 0], g[0, :, 0] * K[:, 4])


def test_host_pipeline_zero_frames():
    plan = _plan()
    pipe = tb.HostPipeline(plan, chunk=4)
    host = torch.zeros((0, 1, CFG2["n_el"], CFG2["n_samples"]), pin_memory=True)
    out = torch.empty((0, 16, 8), pin_memory=True)
    pipe.run(host, out)
    pipe.synchronize()


def test_sweeps_single_depth(ref_vectors):
    eps = float(ref_vectors["eps"])
    m = tb.theta_matrix_sweep([20e-3], tb.ProbeConfig(), tb.Kossoff(0.6), tb.FNumber(1.0),
                              tx_focus_depth=25e-3, window_half_width=eps)
    assert m.values.shape == (1, 1) and m.values[0, 0] == pytest.approx(1.0, rel=1e-9)
    th, loc, glo = tb.error_sweep([20e-3], tb.ProbeConfig(), tb.Kossoff(0.6), tb.FNumber(1.0),
                                  tx_focus_depth=25e-3, window_half_width=eps)
    assert th.shape == loc.shape == glo.shape == (1, 1)
    assert loc[0, 0] == pytest.approx(0.0, abs=1e-20) and glo[0, 0] == pytest.approx(0.0, abs=1e-20)


def test_batch_metrics_zero_batch():
    z = torch.zeros((0, 8), dtype=torch.float64, device=DEV)
    assert tb.batch_errors(z, z, axis=1).shape == (0,)
    assert tb.batch_fwhm(z, 1.0).shape == (0,)


@pytest.mark.parametrize("n", [2048, 4096, 8192])
def test_rf_analytic_writes_stay_inside_the_output(n):
    """Guard bands around the output rows stay untouched (no out-of-bounds stores
    from the register four-step kernels, odd row count)."""
    rows, guard = 3, 4096
    x = torch.randn((rows, n), device=DEV)
    buf = torch.full((rows * n + 2 * guard,), complex(7.0, -7.0), dtype=torch.complex64, device=DEV)
    out = buf[guard: guard + rows * n].view(rows, n)
    tb.rf_analytic(x, "f32", out=out)
    assert bool((buf[:guard] == complex(7.0, -7.0)).all()) and bool((buf[-guard:] == complex(7.0, -7.0)).all())
    assert bool(torch.isfinite(out.real).all()) and bool(torch.isfinite(out.imag).all())


@pytest.mark.parametrize("frames", [1, 9])
def test_das_image_writes_stay_inside_the_output(frames):
    """Guard bands around the image batch stay untouched (ragged grid, partial
    frame batch, deepest-first 1-D grid)."""
    nz, nx, guard = 45, 21, 1024
    plan = _plan(nz, nx)
    rf = torch.randn((frames, 1, CFG2["n_el"], CFG2["n_samples"]), device=DEV)
    buf = torch.full((frames * nz * nx + 2 * guard,), -3.0, device=DEV)
    out = buf[guard: guard + frames * nz * nx].view(frames, nz, nx)
    tb.das_image(rf, plan, out=out)
    assert bool((buf[:guard] == -3.0).all()) and bool((buf[-guard:] == -3.0).all())
    assert bool((out >= 0).all())  # envelopes


@pytest.mark.parametrize("frames", [8, 5])
def test_das_windows_wrapping_the_trace(frames):
    """Pixels whose arrival lies at the very start (tile window below sample 0)
    or end of the trace (window past N - 1): the producer's wrap-around bulk
    copies (periodic indexing, as the analytic-signal gather of the oracle),
    with a full and a partial frame batch, against the oracle."""
    from oracle import das as od
    from tests.setups import plane_t_star
    c = CFG2
    N = c["n_samples"]
    z_end = (N - 1) * c["c"] / (2 * c["fs"])  # 0-degree plane wave: pos = 2 z fs / c
    z = np.concatenate([np.linspace(0.005e-3, 1.0e-3, 40), np.linspace(z_end - 1.5e-3, z_end + 0.2e-3, 56)])
    x = np.linspace(-6e-3, 6e-3, 24)
    rng = np.random.default_rng(3)
    rf = rng.standard_normal((frames, 1, c["n_el"], N)).astype(np.float32)
    plan = tb.plane_wave_plan(n_el=c["n_el"], pitch=c["pitch"], fs=c["fs"], c=c["c"], n_samples=N,
                              x=x, z=z, f_number=c["f_number"])
    img = tb.das_image(torch.as_tensor(rf).to(DEV), plan).cpu().numpy()
    ts = plane_t_star(c, x, z, (0.0,))
    for f in range(frames):
        A = od.analytic_signal(rf[f].astype(np.float64))
        ref = od.das_image_vectorized(A, c["fs"], 0.0, x, z, c["pitch"], c["c"], ts, c["f_number"])
        assert od.rel_l2(img[f], ref) <= 1e-5, f
    assert img[:, -3:].max() == 0.0  # past the end of the trace: np.interp's right = 0
