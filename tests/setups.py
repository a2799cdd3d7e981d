"""Shared test / bench setups: the BASELINE.json configs with the values this
repo pins where the configs leave them open."""
from __future__ import annotations

import numpy as np

from oracle import geom, simulate as osim
from oracle import tidas as otidas

# reference default probe (geometry.py:36-42) and the golden frame "A"
REF_PROBE = dict(n_el=192, pitch=0.2e-3, f0=7e6, fs=50e6, c=1540.0, fbw=0.75)


def ref_frame_A(pts):
    """Reference synthesize_frame(points, focus 25 mm, default probe, Kossoff(0.6))."""
    p = REF_PROBE
    tx_half = geom.ref_aperture_half(25e-3, ("kossoff", 0.6), p["n_el"], p["pitch"], p["c"] / p["f0"])
    tx_xs = (np.arange(-tx_half, tx_half) + 0.5) * p["pitch"]
    xs = geom.element_x(p["n_el"], p["pitch"])
    arr = geom.focused_tx_arrival(pts[:, 0], pts[:, 1], 25e-3, tx_xs, p["c"])
    dist = np.hypot(pts[:, 0][:, None] - xs[None, :], pts[:, 1][:, None])
    sigma = osim.pulse_sigma(p["f0"], p["fbw"])
    n = int(np.ceil(((arr[:, None] + dist / p["c"]).max() + 8 * sigma) * p["fs"])) + 1
    traces = osim.synthesize(pts[:, 0], pts[:, 1], pts[:, 2], n_el=p["n_el"], pitch=p["pitch"],
                             fs=p["fs"], c=p["c"], f0=p["f0"], fbw=p["fbw"], n_samples=n,
                             tx=("focused", 25e-3, tx_xs))
    return traces, tx_xs


# BASELINE.json configs (pinned values: DESIGN.md §Configs)
CFG1 = dict(n_el=64, pitch=0.3e-3, f0=5e6, fs=20e6, c=1540.0, fbw=0.6, n_samples=2048,
            nz=256, nx=128, z=(5e-3, 40e-3), x=(-9.6e-3, 9.6e-3), f_number=1.5)
CFG2 = dict(n_el=128, pitch=0.3e-3, f0=5e6, fs=40e6, c=1540.0, fbw=0.6, n_samples=4096,
            nz=512, nx=256, z=(5e-3, 45e-3), x=(-19.2e-3, 19.2e-3), f_number=1.5,
            n_scat=2000, region_x=(-20e-3, 20e-3), region_z=(5e-3, 45e-3))
CFG3 = dict(CFG2, nz=1024, nx=512, angles=tuple(np.deg2rad(np.linspace(-10, 10, 11))),
            frames=64, n_bright=5)
CFG4 = dict(n_el=128, pitch=0.3e-3, f0=5e6, fs=40e6, c=1540.0, fbw=0.6, n_samples=4096,
            nz=2048, nx=1024, z=(5e-3, 45e-3), x=(-19.2e-3, 19.2e-3), f_number=1.5, taps=129,
            maps=256, density=0.02, neighbourhood=8)
CFG5 = dict(n_el=192, pitch=0.3e-3, f0=5e6, fs=40e6, c=1540.0, fbw=0.6, n_samples=8192,
            nz=1024, nx=1024, z=(5e-3, 60e-3), x=(-28.8e-3, 28.8e-3), f_number=1.5,
            frames=1024, n_scat=4000, target_std=1000.0)


def grid(cfg, nz=None, nx=None):
    nz = nz or cfg["nz"]
    nx = nx or cfg["nx"]
    return np.linspace(*cfg["x"], nx), np.linspace(*cfg["z"], nz)


def speckle_rf(cfg, seed, n_scat=None, angles=(0.0,), n_samples=None):
    """[A][E][N] float64 seeded speckle RF under plane-wave transmits (oracle simulator)."""
    rng = np.random.default_rng(seed)
    sx, sz, a = osim.speckle(rng, n_scat or cfg["n_scat"], cfg["region_x"], cfg["region_z"])
    return np.stack([osim.synthesize(sx, sz, a, n_el=cfg["n_el"], pitch=cfg["pitch"], fs=cfg["fs"],
                                     c=cfg["c"], f0=cfg["f0"], fbw=cfg["fbw"],
                                     n_samples=n_samples or cfg["n_samples"], tx=("plane", ang))
                     for ang in angles]), (sx, sz, a)


def plane_t_star(cfg, x, z, angles=(0.0,)):
    X = np.asarray(x)[None, :]
    Z = np.asarray(z)[:, None]
    return np.stack([geom.plane_wave_expected_arrival(X, Z, a, cfg["n_el"], cfg["pitch"], cfg["c"])
                     for a in angles])
