"""K1 stores only the samples K2 can read (tidas_rf_analytic_range with the
plan's tap range from tidas_das_window_range).

The strong check: the analytic workspace is filled with NaN before das_image,
so any read by K2 outside the stored range would poison the image; images must
equal those of K1's full-row output bitwise."""
import numpy as np
import pytest
import torch

from tests.setups import CFG1, CFG2, CFG3, CFG5, grid

pytestmark = pytest.mark.gpu
tb = pytest.importorskip("paper_2507_15464_b200")
from paper_2507_15464_b200 import imaging  # noqa: E402

DEV = "cuda"


@pytest.mark.parametrize("N,dtype", [(2048, torch.float64), (4096, torch.float32), (4096, torch.int16),
                                     (8192, torch.int16), (8192, torch.float32), (1000, torch.float32)])
def test_rf_analytic_range_stores_only_the_range(N, dtype):
    g = torch.Generator(device=DEV).manual_seed(N)
    rf = torch.randn((5, N), device=DEV, generator=g) * 300
    rf = rf.to(dtype) if dtype != torch.int16 else rf.round().to(torch.int16)
    full = tb.rf_analytic(rf, "f32")
    lo, hi = N // 5 + 3, (3 * N) // 4 + 1
    out = torch.full((5, N), complex(7.0, -7.0), dtype=torch.complex64, device=DEV)
    tb.rf_analytic(rf, "f32", out=out, sample_range=(lo, hi))
    assert torch.equal(out[:, lo:hi + 1], full[:, lo:hi + 1])
    if N in (2048, 4096, 8192):  # the register four-step kernels leave the rest untouched
        sentinel = torch.tensor(complex(7.0, -7.0), dtype=torch.complex64, device=DEV)
        assert bool((out[:, :lo] == sentinel).all()) and bool((out[:, hi + 1:] == sentinel).all())
    with pytest.raises(ValueError):
        tb.rf_analytic(rf, "f32", out=out, sample_range=(hi, lo))


def _plan(cfg, nz, nx, angles=(0.0,), out="envelope"):
    x, zz = grid(cfg, nz, nx)
    return tb.plane_wave_plan(n_el=cfg["n_el"], pitch=cfg["pitch"], fs=cfg["fs"], c=cfg["c"],
                              n_samples=cfg["n_samples"], x=x, z=zz, angles=list(angles), out=out)


def test_cfg2_range_is_the_imaged_depths():
    """cfg2: taps from ~ 2 * 5 mm / c to the deepest pixel's widest receive path."""
    cfg = CFG2
    plan = _plan(cfg, cfg["nz"], cfg["nx"])
    lo, hi = plan.sample_range()
    fs, c = cfg["fs"], cfg["c"]
    assert abs(lo - 2 * 5e-3 / c * fs) < 8
    edge = (45e-3 + np.hypot(45e-3 / 3, 45e-3)) / c * fs  # F#1.5: |x - x_n| < z / 3
    assert edge - 8 < hi < edge + 8
    assert 0 < lo < hi < cfg["n_samples"] - 1


def _nan_workspace_case(cfg, plan, rf):
    ws = imaging.DasWorkspace(plan)
    ws.buf.fill_(float("nan"))
    img = tb.das_image(rf, plan, workspace=ws)
    an = tb.rf_analytic(rf, "f32")  # every sample
    ref = tb.das_from_analytic(an.view(rf.shape[0], plan.n_angles, plan.n_el, plan.n_samples), plan)
    torch.cuda.synchronize()
    assert bool(torch.isfinite(img).all())
    assert torch.equal(img, ref)
    return plan.sample_range()


@pytest.mark.parametrize("case", ["cfg2", "cfg3_coherent", "cfg3_iq", "cfg1_f64rf", "cfg5_i16", "shallow_wrap"])
def test_das_image_never_reads_outside_the_stored_range(case):
    g = torch.Generator(device=DEV).manual_seed(11)
    if case == "cfg2":
        cfg, F = CFG2, 9
        plan = _plan(cfg, 200, 96)
        rf = torch.randn((F, 1, cfg["n_el"], cfg["n_samples"]), device=DEV, generator=g)
    elif case.startswith("cfg3"):
        cfg, F = CFG3, 3
        plan = _plan(cfg, 160, 64, angles=CFG3["angles"], out="coherent" if case == "cfg3_coherent" else "iq")
        rf = torch.randn((F, len(CFG3["angles"]), cfg["n_el"], cfg["n_samples"]), device=DEV, generator=g)
    elif case == "cfg1_f64rf":
        cfg, F = CFG1, 4
        plan = _plan(cfg, cfg["nz"], cfg["nx"])
        rf = torch.randn((F, 1, cfg["n_el"], cfg["n_samples"]), device=DEV, generator=g, dtype=torch.float64)
    elif case == "cfg5_i16":
        cfg, F = CFG5, 2
        plan = _plan(cfg, 128, 96)
        rf = (torch.randn((F, 1, cfg["n_el"], cfg["n_samples"]), device=DEV, generator=g) * 1000).round() \
            .clamp(-32768, 32767).to(torch.int16)
    else:  # pixels at the very start / end of the trace (test_gpu_edges.py): tile windows wrap
        cfg, F = CFG2, 2
        N = cfg["n_samples"]
        z_end = (N - 1) * cfg["c"] / (2 * cfg["fs"])
        z = np.concatenate([np.linspace(0.005e-3, 1.0e-3, 40), np.linspace(z_end - 1.5e-3, z_end + 0.2e-3, 56)])
        plan = tb.plane_wave_plan(n_el=cfg["n_el"], pitch=cfg["pitch"], fs=cfg["fs"], c=cfg["c"], n_samples=N,
                                  x=np.linspace(-6e-3, 6e-3, 24), z=z)
        rf = torch.randn((F, 1, cfg["n_el"], N), device=DEV, generator=g)
    lo, hi = _nan_workspace_case(cfg, plan, rf)
    if case == "shallow_wrap":
        assert (lo, hi) == (0, cfg["n_samples"] - 1)
    else:
        assert hi - lo + 1 < cfg["n_samples"]


# ------------------------------------------------ TIDAS_K1_RF_READY (ABI 6)
@pytest.mark.parametrize("N,dtype,rows", [(2048, torch.float64, 7), (4096, torch.float32, 2048),
                                          (4096, torch.int16, 9), (8192, torch.int16, 1024), (1000, torch.float32, 3)])
def test_rf_ready_flag_same_values_behind_a_busy_kernel(N, dtype, rows):
    """K1 with rf_ready behind a long kernel that is still READING K1's output
    buffer (the situation in das_image's chunk loop): the early loads and
    transforms must not disturb that kernel, and the stores must come out
    bitwise equal to the unflagged call."""
    g = torch.Generator(device=DEV).manual_seed(N + rows)
    rf = torch.randn((rows, N), device=DEV, generator=g) * 300
    rf = rf.to(dtype) if dtype != torch.int16 else rf.round().to(torch.int16)
    plain = tb.rf_analytic(rf, "f32")
    prev = torch.view_as_complex(torch.randn((rows, N, 2), device=DEV, generator=g)).contiguous()
    out = prev.clone()
    acc = torch.zeros((), device=DEV, dtype=torch.float64)
    torch.cuda.synchronize()
    for _ in range(3):
        # a reader of `out` just ahead on the stream, then K1 storing into `out`
        acc += torch.view_as_real(out).double().sum()
        tb.rf_analytic(rf, "f32", out=out, sample_range=(0, N - 1), rf_ready=True)
        assert torch.equal(out, plain)
        out.copy_(prev)
    # the reader saw `prev` every time (the stores waited for it)
    assert float(acc) == pytest.approx(3 * float(torch.view_as_real(prev).double().sum()), rel=1e-12)


def test_das_image_multi_chunk_equals_single_chunk_bitwise():
    """das_image over several chunks (K1 of chunk c + 1 flagged rf_ready behind
    K2 of chunk c) against one chunk holding every frame."""
    cfg = CFG2
    nz, nx, F = 96, 64, 40
    plan = _plan(cfg, nz, nx)
    g = torch.Generator(device=DEV).manual_seed(5)
    rf = torch.randn((F, 1, cfg["n_el"], cfg["n_samples"]), device=DEV, generator=g)
    one = tb.das_image(rf, plan)
    small = _plan(cfg, nz, nx)
    small.chunk_bytes = 8 * cfg["n_el"] * cfg["n_samples"] * 8
    ws = imaging.DasWorkspace(small)
    assert ws.chunk == 8
    for _ in range(3):
        assert torch.equal(tb.das_image(rf, small, workspace=ws), one)
