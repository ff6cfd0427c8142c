"""Tree decode attention and attention-mass accumulation (oracle, test infra).

Decoding of the active leaf "depends exclusively on the ancestor chain of
the active leaf"; attention is over the retained KV of Path(ℓ)
(P:87).  Per active leaf b, layer l and query head g (KV head
h = ⌊g/G⌋, Q24) with scale 1/√d (Q24):
    z_t = q·k_t/√d,  o = Σ_t softmax(z)_t v_t,  LSE = ln Σ_t e^{z_t}
over the visible set V_{b,l,h} = concatenation over Path(ℓ_b), root→leaf,
of the kept positions.  Accumulated attention:
    A[l][h][t] += Σ_{g∈group(h)} exp(z_t − LSE_{b,l,g}).
fp64 throughout (np.float64 matmul as the library primitive).
"""
from __future__ import annotations

import math

import numpy as np


def visible_positions(parent, leaf: int, span_start, kept_of_node) -> np.ndarray:
    """Absolute positions of V_{b,l,h}: Path(ℓ_b) root→leaf, each node's kept
    positions in ascending order.  kept_of_node(i) -> ascending offsets."""
    from .geometry import root_path
    out = []
    for i in root_path(parent, leaf):
        out.extend(int(span_start[i]) + int(t) for t in kept_of_node(i))
    return np.array(out, dtype=np.int64)


def attend(q: np.ndarray, K: np.ndarray, V: np.ndarray):
    """Softmax attention of query rows q [G][d] over keys K [T][d], values
    V [T][d] (fp64).  Returns (o [G][d], lse [G], p [G][T]).

    Max subtraction is the textbook stable evaluation of the same softmax."""
    d = q.shape[-1]
    z = (q @ K.T) / math.sqrt(d)                      # [G][T]
    m = z.max(axis=1, keepdims=True)
    e = np.exp(z - m)
    ssum = e.sum(axis=1, keepdims=True)
    p = e / ssum
    o = p @ V
    lse = (m + np.log(ssum))[:, 0]
    return o, lse, p


def probabilities(q: np.ndarray, K: np.ndarray, lse: np.ndarray) -> np.ndarray:
    """p_t = exp(q·k_t/√d − LSE) for given LSE [G] (the score pass, §8(a) a2)."""
    d = q.shape[-1]
    z = (q @ K.T) / math.sqrt(d)
    return np.exp(z - lse[:, None])
