"""CPU oracle for the MARS scheduling-step hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_2604_26963_b200`` imports this
package; only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may use it, and only as the checker
or as the timed reference CPU path -- never as the product.

The oracle is a from-scratch restatement of the reference's algorithm
(``/root/reference/pkg/src/agentsched``; every function cites the file:line it
follows).  It is *pinned*: ``oracle/make_golden.py`` runs the reference itself
in the dev container and freezes its outputs under ``tests/golden/``; the CPU
test-suite checks this restatement against every one of those fixtures
(byte-identical event logs, known-answer vectors, snapshot-step outputs).
"""
