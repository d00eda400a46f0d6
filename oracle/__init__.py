"""CPU oracle for the NNTile (arXiv 2504.13236) GPT-2 block hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in the product path (the CUDA library, its
Python binding, the block driver) may import, call, link or execute anything
under ``oracle/``.  The only permitted callers are ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg.

Modules
-------
``dense``  plain, untiled fp64 definitions of every step of the path (the
           paper states forward passes only; backward passes are
           the textbook chain rule, reading R18).
``tiled``  the paper's per-tile decomposition written out step by step in fp64
           (tile grid PAPER.md:72-75; softmax two-subroutine form PAPER.md:172-173;
           LayerNorm three steps PAPER.md:162; tiled GEMM PAPER.md:153).

Parity pins: every function is pinned in ``tests/test_oracle_*.py`` against
something other than itself (finite differences, closed forms, torch fp64
library routines, invariants).  One item is "parity unpinned": agreement with
NNTile's own outputs, of which none exist here.

Shares no code with ``paper_2504_13236_b200`` (the product); the seeded input
generators live in ``nnt_inputs.py``, which holds none of the method's
arithmetic.
"""
