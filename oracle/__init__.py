"""PaRO CPU oracle — TEST INFRASTRUCTURE ONLY.

This package is the plain, slow, obviously-correct CPU statement of what the
PaRO (arXiv 2310.06003) data-parallel sync + update step computes.  It exists
to check the CUDA path, never to run in its place:

* only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
  ``cpu_baseline`` / ``--impl reference`` legs may import it;
* it shares no code with ``paper_2310_06003_b200`` (the product) and never
  imports it; the only common dependency is ``paro_synth`` (seeded input
  generators, which hold none of the method's arithmetic).

Citations: ``P:n`` = line n of the paper text, ``S:n`` = line n of
the CPU-program spec.  Readings of silent/garbled passages are the
ones listed in DESIGN.md §3 ("Readings"), labelled R1..Rn below.

Modules
-------
numerics     bf16 RNE, the hop operator, canonical fold, canonical Adam
strategy     the 27 codes, Principle 1 -> 14 PaRO strategies (Table 1)
layout       flat layout, buckets, position-major nested shard map (R1)
collectives  round-synchronous Ring / two-step / HO-Ring / H-Ring simulators
             with per-link byte counters
accounting   Table 2 memory, Table 3 volumes, Eq. 1
step         N-rank strategy step simulator and the unsharded-DP definition

Parity-pin status: every public function here is pinned by a
``-m "not gpu"`` test to something other than itself (paper numbers, closed
forms, brute force, library routines) except where a function's docstring says
"parity unpinned".
"""
