"""Round-2 golden vectors from the reference package (run HERE only; writes
``ref_vectors_r2.npz``). Imports the read-only reference from
/root/reference/pkg/src; nothing at test time reads the reference.

Sets (keys by prefix):

* ``PW_``: the north-star imaging mode of cfg2 (0-degree plane wave, pixel-
  centred Hann F#1.5 apodization) evaluated with the REFERENCE'S OWN primitives
  at 256 seeded pixels of a cfg2 speckle frame: per channel the Hann weight times
  ``das._delay_samples`` (das.py:82-112, linear) of the receive delay
  ``das.target_delays`` (das.py:126-132), summed in channel order, then
  ``metrics.envelope`` (metrics.py:30-34) and np.interp at the plane-wave arrival
  t* = 2 z / c (the reference's ``_envelope_value_at``, das.py:165-178). The RF is
  the oracle simulator's seeded frame rounded to float32 (what the FP32 path
  ingests); the scatterers and seed are stored, not the RF.
* ``NZ_``: a frame with NO leading zeros (reference ``synthesize_frame`` with
  seeded noise, simulate.py:248-251): ``das_value`` / ``das_line`` outputs. The
  drop-in must take its full-trace path (the analytic gather's head-zero
  precondition fails).
* ``CR_``: ``tidas_psf`` crop semantics (tidas.py:336-351): default support,
  a caller-supplied narrower support, the full-length path, and the
  short-segment ValueError.
* ``WS_``: ``window_signals`` (tidas.py:150-168) nonzero bounds and row sums.
* ``TA_``: ``estimate_theta_aligned`` at the inputs of ref test_tidas.py:338.

Usage:  python tests/golden/make_golden_r2.py
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]

# cfg2 (BASELINE.json configs[1]; DESIGN.md §5 pins pitch / grid / region)
CFG2 = dict(n_el=128, pitch=0.3e-3, f0=5e6, fs=40e6, c=1540.0, fbw=0.6, n_samples=4096,
            nz=512, nx=256, z=(5e-3, 45e-3), x=(-19.2e-3, 19.2e-3), f_number=1.5, n_scat=2000,
            region_x=(-20e-3, 20e-3), region_z=(5e-3, 45e-3))
PW_SEED = 2025


def pw_hann_golden(T, vec) -> None:
    from tidas.das import _delay_samples, target_delays
    from tidas.metrics import envelope
    sys.path.insert(0, str(ROOT))
    from oracle import simulate as osim

    c = CFG2
    probe = T.ProbeConfig(element_count=c["n_el"], pitch=c["pitch"], center_frequency=c["f0"],
                          sampling_frequency=c["fs"], sound_speed=c["c"], fractional_bandwidth=c["fbw"])
    rng = np.random.default_rng(PW_SEED)
    sx, sz, amp = osim.speckle(rng, c["n_scat"], c["region_x"], c["region_z"])
    rf = osim.synthesize(sx, sz, amp, n_el=c["n_el"], pitch=c["pitch"], fs=c["fs"], c=c["c"], f0=c["f0"],
                         fbw=c["fbw"], n_samples=c["n_samples"], tx=("plane", 0.0))
    rf = rf.astype(np.float32).astype(np.float64)
    xg, zg = np.linspace(*c["x"], c["nx"]), np.linspace(*c["z"], c["nz"])
    prng = np.random.default_rng(7)
    iz = prng.integers(0, c["nz"], 256)
    ix = prng.integers(0, c["nx"], 256)
    half = c["n_el"] // 2
    idx = np.arange(-half, half)
    xs = (idx + 0.5) * c["pitch"]
    vals = np.empty(256)
    for p, (i, j) in enumerate(zip(iz, ix)):
        x, z = xg[j], zg[i]
        a = z / (2.0 * c["f_number"])
        live = np.abs(xs - x) < a
        total = np.zeros(c["n_samples"])
        for n, w in zip(idx[live], 0.5 * (1.0 + np.cos(np.pi * (xs[live] - x) / a))):
            d = target_delays((x, z), np.array([n]), probe)[0]
            total += w * _delay_samples(rf[n + half], c["fs"], d, "linear")
        env = envelope(T.Trace(total, c["fs"])).samples
        pos = (2.0 * z / c["c"]) * c["fs"]
        vals[p] = float(np.interp(pos, np.arange(c["n_samples"]), env, left=0.0, right=0.0))
    vec.update(PW_seed=PW_SEED, PW_iz=iz, PW_ix=ix, PW_values=vals)
    print("PW+Hann: 256 pixels, max", vals.max())


def no_head_zero_golden(T, vec) -> None:
    p1 = T.ProbeConfig(element_count=64, pitch=0.3e-3, center_frequency=5e6, sampling_frequency=20e6,
                       sound_speed=1540.0, fractional_bandwidth=0.6)
    pts = np.array([(0.0, 15e-3, 1.0), (1e-3, 22e-3, -0.6)])
    frame = T.synthesize_frame(T.ScattererSet.from_points(pts), 20e-3, p1, T.FixedCount(64),
                               noise_amplitude=0.02, rng=np.random.default_rng(11))
    assert np.all(frame.traces[:, 0] != 0.0)  # no head zeros anywhere
    rx = T.FNumber(1.5)
    px = np.linspace(-2e-3, 2e-3, 12)
    pz = np.linspace(12e-3, 25e-3, 12)
    depths = np.linspace(6e-3, 30e-3, 32)
    vec.update(NZ_points=pts, NZ_px=px, NZ_pz=pz, NZ_depths=depths,
               NZ_das_value=np.array([T.das_value(frame, (x, z), p1, rx) for x, z in zip(px, pz)]),
               NZ_das_line=T.das_line(frame, depths, p1, rx))


def crop_golden(T, vec) -> None:
    from tidas.tidas import TimeWindow
    probe, rx, tx = T.ProbeConfig(), T.FNumber(1.0), T.Kossoff(0.6)
    frame = T.synthesize_frame(T.ScattererSet.on_axis([25e-3]), 25e-3, probe, tx)
    psf = T.das_psf(frame, (0.0, 25e-3), probe, rx)
    t_star = T.expected_arrival_time((0.0, 25e-3), frame, probe)
    window = T.fwhm_window(psf, t_star)
    windowed = T.window_signals(frame, window)
    fixed = T.rx_delay_profile(20e-3, T.rx_aperture(25e-3, rx, probe), probe)
    nz = np.flatnonzero(np.any(windowed.traces != 0.0, axis=0))
    s0, s1 = int(nz[0]), int(nz[-1]) + 1
    vec.update(CR_support=np.array([s0, s1]), CR_half_width=window.half_width, CR_center=window.center,
               CR_full=T.tidas_psf(windowed, fixed, 1.3).samples,
               CR_crop=T.tidas_psf(windowed, fixed, 1.3, crop=True).samples,
               CR_crop_narrow=T.tidas_psf(windowed, fixed, 1.3, crop=True, support=(s0 + 4, s1 - 4)).samples)
    try:
        T.tidas_psf(windowed, fixed, 1.3, crop=True, support=(0, 1))
        vec["CR_short_raises"] = False
    except ValueError:
        vec["CR_short_raises"] = True
    # window_signals: nonzero columns and per-row sums of the masked frame; the
    # outside-support windows raise
    vec.update(WS_bounds=np.array([s0, s1]), WS_row_sums=windowed.traces.sum(axis=1))
    raises = []
    for w in (TimeWindow(-1e-6, 1e-7), TimeWindow(frame.times[-1], 1e-6)):
        try:
            T.window_signals(frame, w)
            raises.append(False)
        except ValueError:
            raises.append(True)
    vec["WS_raises"] = np.array(raises)


def theta_aligned_golden(T, vec) -> None:
    """ref test_tidas.py:338 inputs: the reference's own theta (its brute-force
    golden-section check resolves theta only to ~1e-8, see tests/test_gpu_refsuite.py)."""
    from tidas.tidas import TimeWindow, estimate_theta_aligned
    probe, rx, tx = T.ProbeConfig(), T.FNumber(1.0), T.Kossoff(0.6)
    frame = T.synthesize_frame(T.ScattererSet.on_axis([28e-3]), 25e-3, probe, tx)
    w = TimeWindow(T.expected_arrival_time((0.0, 28e-3), frame, probe), 1e-7)
    fixed = T.rx_delay_profile(25e-3, T.rx_aperture(25e-3, rx, probe), probe)
    true = T.rx_delay_profile(28e-3, T.rx_aperture(28e-3, rx, probe), probe)
    vec["TA_theta28"] = estimate_theta_aligned(frame, w, fixed, true)


def main() -> None:
    sys.path.insert(0, str(REF / "src"))
    import tidas as T
    vec = {}
    pw_hann_golden(T, vec)
    no_head_zero_golden(T, vec)
    crop_golden(T, vec)
    theta_aligned_golden(T, vec)
    np.savez_compressed(HERE / "ref_vectors_r2.npz", **vec)
    print("wrote", HERE / "ref_vectors_r2.npz")


if __name__ == "__main__":
    main()
