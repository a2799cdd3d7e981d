"""RF file ingest: save_frame blobs -> one f32 host tensor."""
import numpy as np
import pytest
import torch

import paper_2507_15464_b200 as tb


def _frames(rng, F=3, E=16, N=96):
    return [tb.RfFrame(rng.standard_normal((E, N)), 40e6, 0.0, 20e-3, np.arange(-4, 4)) for _ in range(F)]


def test_read_frames_into_one_tensor(tmp_path, rng):
    frames = _frames(rng)
    bases = []
    for i, f in enumerate(frames):
        tb.save_frame(f, tmp_path / f"f{i}")
        bases.append(tmp_path / f"f{i}")
    t, hdr = tb.read_frames_pinned(bases, pin=False)
    assert t.shape == (3, 1, 16, 96) and t.dtype == torch.float32 and len(hdr) == 3
    for i, f in enumerate(frames):
        assert np.array_equal(t[i, 0].numpy(), f.traces.astype("<f4"))
        assert np.array_equal(tb.load_frame(bases[i]).traces, t[i, 0].numpy().astype(float))


def test_read_frames_rejects_mismatch(tmp_path, rng):
    a, b = _frames(rng, 1)[0], tb.RfFrame(rng.standard_normal((16, 80)), 40e6, 0.0, 20e-3, np.arange(-4, 4))
    tb.save_frame(a, tmp_path / "a")
    tb.save_frame(b, tmp_path / "b")
    with pytest.raises(ValueError):
        tb.read_frames_pinned([tmp_path / "a", tmp_path / "b"], pin=False)
    (tmp_path / "a.f32").write_bytes(b"\0" * 12)
    with pytest.raises(ValueError):
        tb.read_frames_pinned([tmp_path / "a"], pin=False)
    with pytest.raises(ValueError):
        tb.read_frames_pinned([], pin=False)
