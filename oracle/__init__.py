"""TEST INFRASTRUCTURE ONLY — the CPU oracle for the FaaSTube data-passing path.

This package restates, in plain Python/numpy, the algorithms of the reference
simulator ``tubesim`` (``/root/reference/pkg/src/tubesim``) that sit on the
data-passing hot path (SURVEY.md §8a rows a1–a23):

* ``oracle.decisions``      — topology queries, bandwidth matrix, Alg. 1 path
  selection, SLO rate partition, batch triggering, pinned ring, pipeline
  latency model, size classes / histograms / elastic pool policy / migration,
  the two-level data index and ``Dataplane.fetch_plan``.
* ``oracle.stage_arbiter``  — the engine's managed PCIe stage logic
  (``engine.py:116-142, 537-646``) as a replayable state machine.
* ``oracle.host_path``      — the reference's CPU host-memory path
  (``infless_plus``: store = copy into host shared memory, fetch = copy out),
  which defines byte parity (identity) and serves as ``bench.py``'s
  ``cpu_baseline`` / ``--impl reference`` arm.

Parity status: PINNED. ``tests/golden/make_golden.py`` imports the reference
itself (only possible in the build container, where ``/root/reference`` exists)
and records golden decision vectors under ``tests/golden/*.json``;
``tests/test_oracle_golden.py`` checks this oracle against every one of them.
Byte parity is identity (the reference moves no bytes, ``SPEC.md:8``), checked
as uint8 equality.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package. The
product (``paper_2411_01830_b200``) never imports it.
"""
