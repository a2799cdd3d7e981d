"""CPU float64 oracle for the DAS / tiDAS hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg
(``cpu_baseline`` and ``--impl reference``) may import anything from this
package, and only as the checker / the timed CPU reference. The product package
``paper_2507_15464_b200`` never imports it and has no CPU fallback.

Every function restates the reference algorithm (``/root/reference/pkg/src/tidas``)
in plain numpy float64 and cites the file:line it follows. Pinning:

* reference-mode DAS / tiDAS (focused transmit, array-centred boxcar aperture,
  envelope pixel) is pinned against the reference itself: golden vectors in
  ``tests/golden`` produced by ``tests/golden/make_golden.py`` importing the
  reference, including the byte-identical fixture CSVs of
  ``pkg/figures/tests/fixtures``;
* the north-star-only pieces (plane-wave / steered transmit, pixel-centred Hann
  apodization, compounding, int16 ingest, row-kernel builder, row convolution
  and its adjoint) have NO reference counterpart: their parity is "unpinned"
  and rests on this restatement plus identities (adjointness, linearity,
  reduction to the pinned reference mode).
"""
