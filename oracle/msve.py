"""Multi-Signal Value Estimation (oracle, test infrastructure).

PAPER.md §4 "Multi-Signal Value Estimation (MSVE)" P:123-146 and Alg. 1
procedure MSVE: φ_i = [v_i, u_i, a_i],
s_i = clip(σ(θᵀφ_i), 0, 1).  θ carries a bias θ₀ (Q7).  The accumulated
attention feature a_i is the post-close attention mass
paid to block i normalised per query row (Q4, Q5), computed through the
2^24 fixed-point node masses the multi-GPU reduction uses (Q29).
"""
from __future__ import annotations

import math

MASS_SCALE_LOG2 = 24                      # Q29: masses in units of 2^-24
MASS_SCALE = 1 << MASS_SCALE_LOG2


def uncertainty(top_probs, other_mass: float, vocab_size: int) -> float:
    """Eq. 1: H_i = −Σ_w p(w) log p(w); u_i = 1 − H_i/log|𝒱|.

    The optional top-K restriction aggregates the remaining mass into one
    "other" bucket (Q28), which enters the sum as a single term."""
    if vocab_size < 2:
        raise ValueError("|V| must be >= 2")
    h = 0.0
    for p in list(top_probs) + ([other_mass] if other_mass > 0 else []):
        if p < 0:
            raise ValueError("negative probability")
        if p > 0:
            h -= p * math.log(p)
    u = 1.0 - h / math.log(vocab_size)
    return min(1.0, max(0.0, u))


def quantize_mass(m: float) -> int:
    """Q = round-half-even(m · 2^24) as an integer (Q29).  Python's round()
    on a float is round-half-even and exact."""
    return int(round(m * MASS_SCALE))


def row_node_mass(A_row, span_start: int, n: int) -> float:
    """m_{l,h,i} = Σ_{t=a_i}^{b_i} A[l][h][t], all positions of the span, kept
    and evicted alike (evicted A stays frozen).  fp64 sum
    in position order."""
    s = 0.0
    for t in range(span_start, span_start + n):
        s += float(A_row[t])
    return s


def node_mass(A, span_start: int, n: int, rows=None) -> int:
    """Mass_i = Σ_{rows (l,h)} Q(m_{l,h,i}) (exact integer sum, Q29); `rows` restricts the
    sum to a thin slice of (layer, KV head) rows (Q6), default all."""
    total = 0
    L, H = A.shape[0], A.shape[1]
    for l in range(L):
        for h in range(H):
            if rows is not None and (l, h) not in rows:
                continue
            total += quantize_mass(row_node_mass(A[l, h], span_start, n))
    return total


def slice_rows(L: int, H: int, layer_begin: int, kv_head_begin: int, num_layers: int,
               slice_layers: int, slice_kv_heads: int):
    """Local (l, h) rows of the thin slice 𝓛 × 𝓗 ("aggregated over a thin slice of
    heads/layers"): the last `slice_layers` layers of the model and its first
    `slice_kv_heads` KV heads (global indices; 0 = all), as SPEC's default reads
    it.  None when the slice is everything."""
    if not slice_layers and not slice_kv_heads:
        return None
    lo = num_layers - slice_layers if slice_layers else 0
    out = set()
    for l in range(L):
        for h in range(H):
            gl, gh = layer_begin + l, kv_head_begin + h
            if gl >= lo and (not slice_kv_heads or gh < slice_kv_heads):
                out.add((l, h))
    return out


def attention_feature(mass: int, mclose: int, nq: int, num_layers: int,
                      num_q_heads: int) -> float:
    """a_i = clamp((Mass_i − Mclose_i)·2^-24 / (Nq_i·L·Hq), 0, 1); 0 if Nq_i = 0.

    'running mass of attention paid to tokens of block i by later tokens'
    (P:128), post-close only (Q5), normalised per query row (Q4): every query
    row's probabilities sum to 1, so the ratio lies in [0,1]."""
    if nq == 0:
        return 0.0
    x = ((mass - mclose) / MASS_SCALE) / (nq * num_layers * num_q_heads)
    return min(1.0, max(0.0, x))


def sigmoid(x: float) -> float:
    return 1.0 / (1.0 + math.exp(-x))


def msve_score(theta, v: float, u: float, a: float) -> float:
    """s_i = clip(σ(θ₀ + θ_v v_i + θ_u u_i + θ_a a_i), 0, 1) (Alg. 1
    P:502-504; bias per Q7).  fp64; the clip is a formal no-op (Q8)."""
    z = theta[0] + theta[1] * v + theta[2] * u + theta[3] * a
    return min(1.0, max(0.0, sigmoid(z)))
