"""CPU oracle for the sliced + grouped + rehash denoising path.

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_2411_01171_b200`` imports this
package; only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline``
/ ``--impl reference`` legs of ``bench.py`` may use it, and only as the checker
or as the timed CPU baseline -- never as the product path.

It is a numpy restatement of the reference ``sliceflow`` package
(``/root/reference/pkg/src/sliceflow``) plus the three modules the reference
specifies but does not ship (``executor``, ``rehash``, ``harness``:
``SPEC.md:312-512``).  Each function cites the reference file:line it follows.

Pinning: ``tests/golden/make_golden.py`` imports the *real* reference in the
build container and records its outputs (per-kernel vectors, a full toy
denoising run, similarity maps, Algorithm A1 traces, slicer/grouping
structure); ``tests/test_oracle_golden.py`` checks this restatement against
those fixtures.  The graph/weights/plans are host logic shared with the
product package (``paper_2411_01171_b200.unet`` etc.) and are pinned by the
same fixtures.
"""
