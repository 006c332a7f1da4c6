"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct NumPy/SciPy implementation of what the
geometric p-multigrid Laplace solve of arXiv 2009.00705 computes, in FP64.
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import it.  It shares no code
with the CUDA library (``paper_2009_00705_b200``); the only common module is
``workloads`` (seeded input generators, no method arithmetic).

Citation keys: P:n = PAPER.md line n; S:n = SPEC.md line n; O-n / On = the
readings of SURVEY.md §8(c) (restated in DESIGN.md §"Readings").

Modules
-------
refelem   1D rules, triangle nodes, Dubiner/Lagrange bases, prism reference data
sem       geometry factors, element matrices, global numbering, assembly
pmg       transfers, Schwarz smoother, V-cycle (Alg 4.1),
          PDC (Alg 4.2), PCG (Alg 4.3)

Pins: every function is pinned by tests/test_oracle_*.py against closed forms,
brute force or invariants (see DESIGN.md §"Oracle pins").  Parity unpinned:
iteration counts / q versus the paper's tables (different problems).
"""
