"""ORACLE -- test infrastructure, NOT product code.

A plain, slow, obviously-correct CPU implementation of what the hot path
computes, written from PAPER.md (arXiv 2503.05248) and the readings listed in
DESIGN.md "Readings of the paper".  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import,
call, link or execute anything here.  It shares no code, headers, constants or
helpers with the CUDA library in ``paper_2503_05248_b200/``; the only common
dependency is ``synth/`` (seeded input generators with none of the method's
arithmetic).

Modules (each function cites the passage it follows):
* ``attention``  -- O1 paged decode attention, fp64, two-pass full softmax (C, ``attention.c``)
* ``allocator``  -- O2 page allocator (lowest-free-page-first, all-or-nothing)
* ``stats``      -- O3 batch statistics record (integer definitions of §8(a)-S4)
* ``chance``     -- O4 Eqs. 7-11: theta, overflow probability, largest feasible b
* ``policy``     -- O5 Algorithm 1, O6 Algorithm 2, the min-combination
* ``engine``     -- O7 continuous-batching replay (S1 -> S7) on logged step times
* ``model``      -- O8 full decode step of a Llama-2-shaped decoder (NEXT row 3), fp64

Parity status per function is in DESIGN.md "Oracle pins".
"""
