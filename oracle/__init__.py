"""CPU oracle for the TF-Replicator data-parallel hot path. TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg may import this package, and only as the checker (or as
the timed reference CPU arm). The product path (``paper_1902_00465_b200``) never
imports it and fails loudly when its CUDA library is missing.

Parity status: PINNED. ``tests/golden/*.npz`` were produced by running the
reference package itself (``/root/reference/pkg/src/replicator``, imported in the
build container by ``oracle/make_golden.py``) and ``tests/test_oracle.py`` checks
this restatement against every fixture plus the SPEC known-answer tests.
"""
