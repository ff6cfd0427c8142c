"""Token-extractive selection (oracle, test infrastructure).

PAPER.md §4 "Execution" and Alg. 1 procedure Evict
(P:512-520): keep the block tail 𝒯_i and the top-m_i heavy
hitters 𝓗_i by accumulated attention A_i(t), m_i = k_i − |𝒯_i|;
if k_i ≤ L_tail return the last k_i positions.  Readings:
candidates are the currently kept non-tail positions (Q2); the order is the
key ⟨f32 A, position⟩ descending (Q3); per-(layer, KV head) rows (Q1).
"""
from __future__ import annotations

import numpy as np


def f32_bits(a: float) -> int:
    """Orderable bits of a non-negative f32 value; −0 canonicalised to +0 (Q3)."""
    x = np.float32(a)
    if x == 0:
        return 0
    if not np.isfinite(x) or x < 0:
        raise ValueError("A must be finite and non-negative (ARBOR_ERR_INVARIANT)")
    return int(np.array([x], dtype=np.float32).view(np.uint32)[0])


def key(a_f32: float, offset: int):
    """key(t) = (f32 A(t), t): larger A first, on equal A the more recent
    position first (Q3)."""
    return (f32_bits(a_f32), int(offset))


HEAVY, TAIL, SINKS_TAIL = 0, 1, 2   # intra-block rules (arbor_select_mode; P:660-675 ablation)


def rank_key(mode: int, a_f32: float, t: int, n_sinks: int, is_root: bool = False):
    """Order of the non-tail candidates, descending.  Global sinks 𝒮 — the first n_sinks
    positions of the initial prompt = the root block (Q22) — come first in HEAVY
    ("plus global sinks 𝒮 shared across all blocks") and SINKS_TAIL; then ⟨A, t⟩ for
    the method's heavy hitters (Q3), t alone (recency) for Sinks + Tail and
    Tail-only (Tail-only keeps no sinks).  The root is on Path* and pinned in the
    default policy, so sinks only matter when it can be evicted (k_protect > 0)."""
    sink = 1 if (is_root and t < n_sinks and mode != TAIL) else 0
    if mode == HEAVY:
        return (sink,) + key(a_f32, t)
    return (sink, 0, int(t))


def retained_set(kept, n: int, k_app: int, l_tail: int, A_node_f32, mode: int = HEAVY,
                 n_sinks: int = 0, is_root: bool = False):
    """Alg. 1 Evict for one (row, node).

    kept: within-node offsets currently retained (C, any order);
    A_node_f32: f32 accumulated attention indexed by within-node offset (HEAVY only).
    Returns the new ascending retained offsets ℛ with |ℛ| = k_app."""
    kept = [int(x) for x in kept]
    assert 0 <= k_app <= len(kept)
    tl = min(l_tail, n)
    if k_app <= tl:                           # Alg. 1: the last k_i
        R = list(range(n - k_app, n))
        assert set(R) <= set(kept)
        return R
    tail = list(range(n - tl, n))             # 𝒯_i
    assert set(tail) <= set(kept)
    m = k_app - tl                            # m_i = k_i − |𝒯_i|
    cand = [t for t in kept if t < n - tl]
    ranked = sorted(cand, key=lambda t: rank_key(mode, A_node_f32[t] if mode == HEAVY else 0.0,
                                                 t, n_sinks, is_root), reverse=True)
    heavy = ranked[:m]                        # Top-m_i by A_i(t), or the variant's order
    return sorted(tail + heavy)


def trim_prefix(tail, heavy, k: int, A_node_f32):
    """SPEC S:402 trim oracle: sort tail ∪ heavy by (is_tail desc, A desc,
    pos desc) and keep the first k ('prioritize tail tokens first and
    then heavy hitters by A_i(t)')."""
    T = set(tail)
    allp = sorted(set(tail) | set(heavy),
                  key=lambda t: (1 if t in T else 0, f32_bits(A_node_f32[t]), t),
                  reverse=True)
    return sorted(allp[:k])
