"""Seeded randomised plans through the public DAS path (K1 + K2) against the
float64 oracle. Plane-wave plans (FP32): array sizes, trace lengths (powers of two and Bluestein
lengths), sampling rates, ragged pixel grids placed anywhere on the trace
(windows that wrap or exceed the staging boxes), steered transmits, F-numbers,
the three output modes, RF dtypes and frame counts that leave partial frame
batches. Table plans (random arrival tables, t0 != 0, the reference's boxcar
or Hann apertures, FP32 and FP64) against the per-pixel oracle. Tolerance: the
north-star 1e-5 relative L2 for FP32, 1e-11 for FP64 (absolute, of the
reference scale, when the reference image is empty). The first version of this
file found two bugs: odd trace lengths staged with 16-byte copies, and a pixel
marked inactive for one steering angle staying inactive for the next."""
import numpy as np
import pytest
import torch

import paper_2507_15464_b200 as tb
from oracle import das as od
from oracle import geom

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _case(seed):
    rng = np.random.default_rng(1000 + seed)
    n_el = int(rng.choice([16, 32, 48, 64, 96, 128]))
    pitch = float(rng.uniform(0.15e-3, 0.4e-3))
    fs = float(rng.choice([20e6, 31.25e6, 40e6, 50e6]))
    c = 1540.0
    n = int(rng.choice([512, 1000, 1024, 2048, 2285, 4096]))
    z_max = (n - 1) * c / (2 * fs) * float(rng.uniform(0.3, 1.15))  # may run past the trace end
    z0 = float(rng.uniform(0.0, 0.3)) * z_max
    nz, nx = int(rng.integers(1, 70)), int(rng.integers(1, 40))
    z = np.sort(rng.uniform(z0, z_max, nz)) if rng.random() < 0.3 else np.linspace(z0 + 1e-5, z_max, nz)
    half_w = float(rng.uniform(0.2, 1.0)) * n_el * pitch / 2
    x = np.linspace(-half_w, half_w, nx) + float(rng.uniform(-1, 1)) * pitch
    n_ang = int(rng.integers(1, 4))
    angles = tuple(np.deg2rad(rng.uniform(-20, 20, n_ang)))
    f_number = float(rng.uniform(0.7, 3.0))
    out = str(rng.choice(["envelope", "coherent", "iq"]))
    dtype = [np.float32, np.int16, np.float64][int(rng.integers(0, 3))]
    frames = int(rng.integers(1, 12))
    rf = rng.standard_normal((frames, n_ang, n_el, n)) * (1000.0 if dtype == np.int16 else 1.0)
    rf = np.rint(rf).astype(dtype) if dtype == np.int16 else rf.astype(dtype)
    return dict(n_el=n_el, pitch=pitch, fs=fs, c=c, n=n, x=x, z=z, angles=angles, f_number=f_number,
                out=out, rf=rf)


@pytest.mark.parametrize("seed", range(40))
def test_das_random_plan_vs_oracle(seed):
    k = _case(seed)
    plan = tb.plane_wave_plan(n_el=k["n_el"], pitch=k["pitch"], fs=k["fs"], c=k["c"], n_samples=k["n"],
                              x=k["x"], z=k["z"], angles=k["angles"], f_number=k["f_number"], out=k["out"])
    img = tb.das_image(torch.as_tensor(k["rf"]).to(DEV), plan).cpu().numpy()
    X = np.asarray(k["x"])[None, :]
    Z = np.asarray(k["z"])[:, None]
    ts = np.stack([geom.plane_wave_expected_arrival(X, Z, a, k["n_el"], k["pitch"], k["c"]) for a in k["angles"]])
    for f in range(k["rf"].shape[0]):
        A = np.stack([od.analytic_signal(k["rf"][f, a].astype(np.float64)) for a in range(len(k["angles"]))])
        ref = od.das_image_vectorized(A, k["fs"], 0.0, k["x"], k["z"], k["pitch"], k["c"], ts, k["f_number"],
                                      out=k["out"])
        scale = max(float(np.abs(ref).max()), 1e-30)
        err = float(np.linalg.norm(img[f] - ref) / max(np.linalg.norm(ref), 1e-30))
        assert err <= 1e-5 or float(np.abs(img[f] - ref).max()) <= 1e-5 * scale, \
            (seed, f, err, plan.window(), k["n"], k["out"])


def _table_case(seed):
    """Random arrival tables (t* anywhere on the trace, per transmit), t0 != 0,
    the reference's array-centred boxcar apertures or Hann, either precision."""
    rng = np.random.default_rng(5000 + seed)
    n_el = int(rng.choice([8, 16, 32, 64]))
    pitch = float(rng.uniform(0.15e-3, 0.4e-3))
    fs = float(rng.choice([20e6, 40e6]))
    c = 1540.0
    n = int(rng.choice([256, 700, 1024, 2048]))
    t0 = float(rng.uniform(-5, 5)) / fs
    nz, nx, n_ang = int(rng.integers(1, 14)), int(rng.integers(1, 9)), int(rng.integers(1, 3))
    z = np.sort(rng.uniform(2e-3, (n - 1) * c / (2 * fs), nz))
    x = np.sort(rng.uniform(-n_el * pitch / 2, n_el * pitch / 2, nx))
    # t*: the receive leg z / c plus a transmit leg in [0, 2 z / c), with some
    # pixels pushed off either end of the trace
    t_star = (z[None, :, None] / c) * (1.0 + rng.uniform(0.0, 2.0, (n_ang, nz, nx)))
    t_star += rng.choice([0.0, 0.0, 0.0, -1.0, 1.0], (n_ang, nz, nx)) * n / fs * 0.6
    if rng.random() < 0.5:
        rule = ("fnumber", float(rng.uniform(0.8, 3.0)))
        half = np.array([geom.ref_aperture_half(zz, rule, n_el, pitch, c / 5e6) for zz in z], np.int32)
        aperture, oracle_ap = ("ref", half), ("ref", rule, c / 5e6)
    else:
        f_number = float(rng.uniform(0.8, 3.0))
        aperture, oracle_ap = ("hann", f_number), ("hann", f_number)
    prec = "f64" if rng.random() < 0.5 else "f32"
    out = str(rng.choice(["envelope", "coherent", "iq"]))
    frames = int(rng.integers(1, 10))
    rf = rng.standard_normal((frames, n_ang, n_el, n))
    return dict(n_el=n_el, pitch=pitch, fs=fs, c=c, n=n, t0=t0, x=x, z=z, t_star=t_star, aperture=aperture,
                oracle_ap=oracle_ap, prec=prec, out=out, rf=rf)


@pytest.mark.parametrize("seed", range(16))
def test_das_random_table_plan_vs_oracle(seed):
    k = _table_case(seed)
    plan = tb.table_plan(n_el=k["n_el"], pitch=k["pitch"], fs=k["fs"], c=k["c"], n_samples=k["n"], x=k["x"],
                         z=k["z"], t_star=k["t_star"], aperture=k["aperture"], out=k["out"], prec=k["prec"],
                         t0=k["t0"])
    rf = torch.as_tensor(k["rf"].astype(np.float64 if k["prec"] == "f64" else np.float32)).to(DEV)
    img = tb.das_image(rf, plan).cpu().numpy()
    tol = 1e-11 if k["prec"] == "f64" else 1e-5
    for f in range(k["rf"].shape[0]):
        A = np.stack([od.analytic_signal(k["rf"][f, a]) for a in range(k["rf"].shape[1])])
        ref = od.das_image(A, k["fs"], k["t0"], k["x"], k["z"], k["pitch"], k["c"], k["t_star"], k["oracle_ap"],
                           out=k["out"])
        scale = max(float(np.abs(ref).max()), 1e-30)
        err = float(np.linalg.norm(img[f] - ref) / max(np.linalg.norm(ref), 1e-30))
        assert err <= tol or float(np.abs(img[f] - ref).max()) <= tol * scale, (seed, f, err, k["prec"], k["out"])
