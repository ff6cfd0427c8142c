"""Event-driven controller oracle: Alg. 2 (PAPER.md Appendix; §3).

TEST INFRASTRUCTURE ONLY (tests/, smoke() and bench.py's cpu_baseline may use it; the
product path never does).  Plain Python over `ArborOracle` (oracle/state.py), following the
pseudocode line by line:

  Boundary(i)      l.3-4   ScoreAllocEvict(i): Eqs. 2-3 (TAE) for block i only,
                           "evict the earliest n_i − k_i tokens of that block only"
  Transition(ℓ)    l.5-21  Path* ← RootToLeaf(ℓ); every i ∈ Path* with k_i < n_i is
                           rehydrated (k_i ← n_i); every j ∉ Path* gets k_j^new = TAE(...)
                           and is evicted only if k_j^new < k_j
  Pressure         l.22-30 every j ∉ Path*: k_j ← TAE(...) and evict; while Σ k > 𝓑: the
                           lowest-Priority off-path block loses one token (floor K_min)
  waterline        l.31-33 raise Pressure when Σ_i k_i ≥ 𝓑 − δ

Readings ("f1 controller"):
  * TAE at Boundary / Transition = Eqs. 2-3 (allocation mode STATIC); at Pressure the
    allocation is the bundle's mode: STATIC_DRAIN is Alg. 2 literally (Eqs. 2-3 then the
    unit-step drain in Priority order, Q16), WATERFILL is the budget-exact optimisation view
     — both end with Σ k ≤ 𝓑.
  * Retained sets only shrink outside rehydration (Q17): an evict applies min(k_cur, k_new).
  * At most one pending Pressure; it is handled right after the event (or
    token step) that raised it.
  * Scores s_i are the MSVE scores of the last scoring pass (Alg. 1; passed in).
  * Parity unpinned: the paper gives no δ; 𝓑 − δ is an input.
"""
from __future__ import annotations

from . import tae

BOUNDARY, TRANSITION, PRESSURE = "boundary", "transition", "pressure"


class ControllerOracle:
    def __init__(self, orc, budget: int, delta: int, pressure_mode=None):
        self.orc = orc
        self.budget = int(budget)
        self.delta = int(delta)
        mode = orc.params["alloc_mode"] if pressure_mode is None else pressure_mode
        # a STATIC bundle cannot meet a budget: Alg. 2's Pressure is STATIC + drain
        self.pressure_mode = tae.MODE_STATIC_DRAIN if mode == tae.MODE_STATIC else mode
        self.pending = False
        self.log = []        # (event, node or -1, Σ k after)

    # ------------------------------------------------------------ helpers
    def total(self) -> int:
        """M ∝ Σ_{i∈V} k_i; open blocks hold their current length."""
        return sum(self.orc.k_cur(i) for i in range(len(self.orc.n)))

    def _static_targets(self, tree, s):
        d, dist, on_path = self.orc.geometry(tree)
        st, k, _ = tae.allocate(tae.MODE_STATIC, s, d, dist, on_path, self.orc.open, self.orc.n,
                                self.orc.params, self.budget)
        assert st == tae.STATUS_OK
        return k

    # ------------------------------------------------------------ Alg. 2 branches
    def boundary(self, tree, i: int, s, A_f32=None):
        """l.3-4: ScoreAllocEvict(i) — block i only."""
        assert not self.orc.open[i], "Boundary refers to a just-closed block"
        k = self._static_targets(tree, s)
        target = [self.orc.n[j] for j in range(len(self.orc.n))]   # others: unchanged
        target[i] = k[i]
        self.orc.evict(tree, target, A_f32=A_f32)
        self.log.append((BOUNDARY, i, self.total()))

    def transition(self, tree, s, A_f32=None):
        """l.5-21: pin and rehydrate Path*, re-target the off-path blocks (shrink only)."""
        _, _, on_path = self.orc.geometry(tree)
        path = [x for x in range(len(self.orc.n)) if on_path[x] and not self.orc.open[x]]
        protect = int(self.orc.params.get("k_protect", 0))
        if protect:   # invariant (i) with the high floor: only blocks below it
            path = [x for x in path if self.orc.k_cur(x) < min(self.orc.n[x], protect)]
        self.orc.rehydrate(path)
        k = self._static_targets(tree, s)
        self.orc.evict(tree, k, A_f32=A_f32)
        self.log.append((TRANSITION, -1, self.total()))

    def pressure(self, tree, s, A_f32=None):
        """l.22-30: reallocate the off-path blocks to the budget, evict."""
        k = self.orc.allocate(tree, s, self.budget, mode=self.pressure_mode)
        self.orc.evict(tree, k, A_f32=A_f32)
        self.pending = False
        self.log.append((PRESSURE, -1, self.total()))

    def waterline(self) -> bool:
        """l.31-33: raise Pressure iff Σ k ≥ 𝓑 − δ and none is pending."""
        if not self.pending and self.total() >= self.budget - self.delta:
            self.pending = True
            return True
        return False
