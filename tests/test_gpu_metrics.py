"""On-device batched metrics vs the oracle (pinned by golden
reference vectors in tests/test_oracle.py)."""
import numpy as np
import pytest
import torch

import paper_2507_15464_b200 as tb
from oracle import metrics as om
from oracle import theta as oth

pytestmark = pytest.mark.gpu
DEV = "cuda"


def test_batch_errors_frames_lines_windows(rng):
    ref = rng.standard_normal((3, 40, 24))
    cand = ref + 0.05 * rng.standard_normal(ref.shape)
    for dt in (torch.float64, torch.float32):
        r, c = torch.as_tensor(ref, dtype=dt, device=DEV), torch.as_tensor(cand, dtype=dt, device=DEV)
        rn, cn = r.double().cpu().numpy(), c.double().cpu().numpy()
        g = tb.batch_errors(r, c).cpu().numpy()
        want = [oth.global_error(rn[f].ravel(), cn[f].ravel()) for f in range(3)]
        np.testing.assert_allclose(g, want, rtol=1e-12)
        lines = tb.batch_errors(r, c, axis=1).cpu().numpy()  # depth lines [F][nx]
        want = [[oth.global_error(rn[f, :, x], cn[f, :, x]) for x in range(24)] for f in range(3)]
        np.testing.assert_allclose(lines, want, rtol=1e-12)
        loc = tb.batch_errors(r, c, axis=1, window=(5, 17)).cpu().numpy()
        want = [[oth.local_error(rn[f, :, x], cn[f, :, x], 5, 17) for x in range(24)] for f in range(3)]
        np.testing.assert_allclose(loc, want, rtol=1e-12)
    z = torch.zeros((2, 8), dtype=torch.float64, device=DEV)
    assert torch.isnan(tb.batch_errors(z, z)).all()
    with pytest.raises(ValueError):
        tb.batch_errors(z, z, axis=1, window=(4, 4))


def test_batch_fwhm_vs_oracle_and_golden(ref_vectors, rng):
    env = torch.as_tensor(ref_vectors["G_env_rows"], device=DEV)
    w = tb.batch_fwhm(env, 50e6).cpu().numpy()
    np.testing.assert_allclose(w, ref_vectors["G_half_widths"], rtol=1e-13)
    # depth lines of images (axis 1), with degenerate lines -> NaN
    t = np.linspace(-1, 1, 65)
    imgs = np.exp(-((t[None, :, None] - rng.uniform(-0.5, 0.5, (2, 1, 7))) ** 2) / 0.02) * \
        rng.uniform(0.5, 2.0, (2, 1, 7))
    imgs[0, :, 3] = -1.0                     # non-positive maximum
    imgs[1, :, 5] = np.linspace(0, 1, 65)    # maximum at the edge: no right crossing
    got = tb.batch_fwhm(torch.as_tensor(imgs, dtype=torch.float32, device=DEV), 1e3, axis=1).cpu().numpy()
    x32 = imgs.astype(np.float32).astype(np.float64)
    for f in range(2):
        for x in range(7):
            try:
                want = om.width_at_half_max(x32[f, :, x], 1e3)
            except ValueError:
                assert np.isnan(got[f, x])
                continue
            assert got[f, x] == pytest.approx(want, rel=1e-12)


def test_batch_fwhm_of_rf_envelope(ref_vectors):
    from oracle import das as od
    rows = ref_vectors["G_env_rows"]  # already envelopes: use them as "RF" with known envelope
    got = tb.batch_fwhm(torch.as_tensor(rows, device=DEV), 50e6, envelope=True).cpu().numpy()
    want = [om.width_at_half_max(od.envelope(r), 50e6) for r in rows]
    np.testing.assert_allclose(got, want, rtol=1e-10)


def test_batch_sidelobe_stats_vs_golden_and_oracle(ref_vectors, rng):
    d = np.linspace(5e-3, 40e-3, 64)
    sc = [12e-3, 25e-3, 31e-3]
    line = torch.as_tensor(ref_vectors["A_tidas_line"], device=DEV)[None]
    refl = torch.as_tensor(ref_vectors["A_das_line"], device=DEV)[None]
    db, rel = tb.batch_sidelobe_stats(line, d, sc, 3, reference=refl)
    np.testing.assert_allclose([db.item(), rel.item()], ref_vectors["G_sidelobe"], rtol=1e-12)
    imgs = np.abs(rng.standard_normal((2, 64, 5)))
    got, _ = tb.batch_sidelobe_stats(torch.as_tensor(imgs, device=DEV), d, sc, 2, axis=1)
    for f in range(2):
        for x in range(5):
            assert got[f, x].item() == pytest.approx(om.sidelobe_stats(imgs[f, :, x], d, sc, 2)[0], rel=1e-12)
    with pytest.raises(ValueError):
        tb.batch_sidelobe_stats(line, d, [50e-3], 3)
