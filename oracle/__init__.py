"""ArborKV CPU oracle — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU implementation of what ArborKV's
per-step KV-eviction path computes (PAPER.md = /root/reference/PAPER.md,
cited as P:<line>; SURVEY.md §8(c) readings cited as Q<n>).  Floating point
is fp64 (numpy); the budget allocation is exact rational arithmetic
(``fractions.Fraction`` / Python ints).  Each function cites the passage it
follows, in the paper's order and notation.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import anything under
``oracle/``.  The product path (``paper_2605_22106_b200``) never imports it,
and this package never imports the product: they share no code.  The only
shared module is ``synth/`` (seeded input generators, no method arithmetic).

Parity status of each function is listed in DESIGN.md §"Oracle pins".
Parity unpinned: the MSVE weight *values* θ (never published) — any θ
is accepted, only the functional form is pinned.
"""
from . import geometry, msve, tae, select, attention, state  # noqa: F401
from .state import ArborOracle  # noqa: F401
