"""Tree-Aware Eviction budget allocation (oracle, test infrastructure).

PAPER.md §4 "Tree-Aware Eviction (TAE)" Eq. 2 and Eq. 3
(P:156-166), Alg. 1 procedure TAE, the "Optimization view"
(min Σ −w_i log k_i s.t. Σ k_i ≤ 𝓑, KKT k*_i = min{n_i, w_i/λ}),
and Alg. 2's Pressure drain.

Three modes (include/arbor.h arbor_alloc_mode):
  WATERFILL     the optimisation view with the floors of Eq. 3 as box
                constraints, solved exactly (Q12), integerised by largest
                remainder so that Σ k = 𝓑.
  STATIC        Eqs. 2-3 directly (no budget guarantee).
  STATIC_DRAIN  STATIC, then Alg. 2's `while Σk > 𝓑: k_j ← max(K_min, k_j−1)`
                on argmin Priority (Priority = W_j, Q16).

All arithmetic after the one fp64 weight product is exact (Python ints and
fractions.Fraction); the waterfill is written as its plain definition: find
λ > 0 with Σ_j clamp(W_j/λ, f_j, n_j) = 𝓑' by scanning the sorted
breakpoints.
"""
from __future__ import annotations

import math
from fractions import Fraction

WEIGHT_SCALE_LOG2 = 24          # Q29: W_j = round(w_j · 2^24)
WEIGHT_SCALE = 1 << WEIGHT_SCALE_LOG2
EPS_FLOOR = 1e-9                # Q10: ⌊x + 1e-9⌋

MODE_WATERFILL, MODE_STATIC, MODE_STATIC_DRAIN, MODE_STREAM = 0, 1, 2, 3

STATUS_OK = 0
STATUS_INFEASIBLE = 3


def eps_floor(x: float) -> int:
    """⌊x⌋ of Eq. 3 read as ⌊x + 10⁻⁹⌋ (Q10): r=0.29, n=100 gives 29, not 28."""
    return int(math.floor(x + EPS_FLOOR))


def tail_len(n: int, l_tail: int) -> int:
    """|𝒯_i| = min{L_tail, n_i}."""
    return min(l_tail, n)


def keep_count(r: float, n: int, k_min: int, l_tail: int) -> int:
    """Eq. 3: k = min{n, max(K_min, |𝒯|, ⌊r n⌋)} (Alg. 1's
    max{K_min, L_tail, ⌊rn⌋} then min{k,n} is the same function, Q11)."""
    return min(n, max(k_min, tail_len(n, l_tail), eps_floor(r * float(n))))


def floor_count(n: int, k_min: int, l_tail: int, r_min: float) -> int:
    """Per-block floor f_j = min(n, max(K_min, min(L_tail,n), ⌊r_min·n⌋)):
    invariant (ii) plus Eq. 2's r ≥ r_min (Q13)."""
    return min(n, max(k_min, tail_len(n, l_tail), eps_floor(r_min * float(n))))


def exp_table(lmbda: float, size: int) -> list:
    """E[x] = exp(−λ·x) for integer x (the e^{−λ_d d_i}, e^{−λ_Δ Δ_i} factors of
    Eq. 2); host libm (Q9)."""
    return [math.exp(-lmbda * x) for x in range(size)]


def powi(s: float, gamma: float) -> float:
    """s^γ: repeated multiplication for integer γ (Q9), else exp(γ·log s)."""
    if float(gamma).is_integer() and 0 <= gamma <= 64:
        p = 1.0
        for _ in range(int(gamma)):
            p = p * s
        return p
    if s <= 0.0:
        return 0.0
    return math.exp(gamma * math.log(s))


def weight(s: float, depth: int, dist: int, off_path: bool, gamma: float, eta: float,
           E_d: list, E_D: list) -> float:
    """Value-geometry weight w = s^γ · e^{−λ_d d} · e^{−λ_Δ Δ} times the
    off-path discount η^{𝟙(i∉Path*)} of Eq. 2; strictly left-to-right
    fp64 products."""
    w = powi(s, gamma)
    w = w * E_d[depth]
    w = w * E_D[dist]
    if off_path:
        w = w * eta
    return w


def quantize_weight(w: float) -> int:
    """W = round-half-even(w · 2^24) (Q29)."""
    if not (w >= 0.0) or w > 65536.0:
        raise ValueError("weight out of range")
    return int(round(w * WEIGHT_SCALE))


def box_waterfill(W, f, n, budget):
    """Relaxed allocation of the optimisation view with the floors
    as box constraints (Q12): k*_j = clamp(W_j/λ, f_j, n_j), Σ k*_j = budget.

    Requires every W_j > 0 and Σ n_j > budget ≥ Σ f_j.  Returns
    (k_star: list[Fraction], active: list[bool], Num, Den) where on the active
    set k*_j = W_j·Num/Den (λ = Den/Num)."""
    m = len(W)
    assert all(w > 0 for w in W)
    assert sum(n) > budget >= sum(f)

    def S(lam: Fraction) -> Fraction:
        return sum(min(max(Fraction(W[j]) / lam, Fraction(f[j])), Fraction(n[j]))
                   for j in range(m))

    bps = {Fraction(W[j], n[j]) for j in range(m)}
    bps |= {Fraction(W[j], f[j]) for j in range(m) if f[j] > 0}
    bps = sorted(bps)
    # S is nonincreasing in λ; at the smallest breakpoint every node is capped
    beta = None
    for b in bps:
        if S(b) >= budget:
            beta = b
    assert beta is not None
    # classification on the open interval just above β
    capped = [Fraction(W[j], n[j]) > beta for j in range(m)]
    floored = [(not capped[j]) and f[j] > 0 and Fraction(W[j], f[j]) <= beta
               for j in range(m)]
    active = [not capped[j] and not floored[j] for j in range(m)]
    num = budget - sum(n[j] for j in range(m) if capped[j]) \
        - sum(f[j] for j in range(m) if floored[j])
    den = sum(W[j] for j in range(m) if active[j])
    k_star = []
    for j in range(m):
        if capped[j]:
            k_star.append(Fraction(n[j]))
        elif floored[j]:
            k_star.append(Fraction(f[j]))
        else:
            k_star.append(Fraction(W[j] * num, den))
    return k_star, active, num, den


def integerize(W, f, n, k_star, active, num, den, ids):
    """base = ⌊k*⌋ on the active set, then the leftover
    tokens go one each to the active nodes with the largest remainder
    (W_j·Num mod Den), ties → larger W_j, then smaller node id."""
    k = []
    for j in range(len(W)):
        k.append(int(k_star[j]) if not active[j] else (W[j] * num) // den)
    target = sum(k_star)
    assert target.denominator == 1
    leftover = int(target) - sum(k)
    if leftover:
        cand = [j for j in range(len(W)) if active[j]]
        cand.sort(key=lambda j: (-((W[j] * num) % den), -W[j], ids[j]))
        for j in cand[:leftover]:
            k[j] += 1
    return k


def proportional_slack(f, n, R, ids):
    """Saturation rule for zero-weight nodes:
    k_j = f_j + ⌊(n_j−f_j)·R/S⌋ with S = Σ(n_j−f_j), leftover by largest
    remainder ((n_j−f_j)·R mod S), ties → smaller node id."""
    S = sum(n[j] - f[j] for j in range(len(n)))
    if S == 0:
        return list(f)
    k = [f[j] + ((n[j] - f[j]) * R) // S for j in range(len(n))]
    leftover = sum(f) + R - sum(k)
    cand = sorted(range(len(n)), key=lambda j: (-(((n[j] - f[j]) * R) % S), ids[j]))
    for j in cand[:leftover]:
        k[j] += 1
    return k


def stream_targets(parent, leaf: int, is_open, n, n_sinks: int, budget: int):
    """The sequence-flattened StreamingLLM analogue (the baselines are adapted to
    ToT "by treating the currently active search path as the streaming sequence"; SPEC
    S:626 SeqFlat with no heavy hitters): the active path root → ℓ is one token stream that
    keeps its global sinks (the root's first n_sinks tokens) and its most recent
    W = 𝓑 − Σ_open n − |sinks| tokens; blocks off the path are outside the stream (k = 0).
    Open blocks stay pinned.  Returns (status, k, min_feasible)."""
    N = len(n)
    k = [n[j] if is_open[j] else 0 for j in range(N)]
    s0 = min(n_sinks, n[0]) if not is_open[0] else 0
    need = sum(n[j] for j in range(N) if is_open[j]) + s0
    if budget < need:
        return STATUS_INFEASIBLE, None, need
    rem = budget - need
    path = []
    x = leaf
    while x >= 0:
        path.append(x)
        x = parent[x]
    for x in path:                      # leaf first: the most recent tokens
        if is_open[x]:
            continue
        w = min(n[x], rem)
        rem -= w
        k[x] = min(n[x], s0 + w) if x == 0 else w
    return STATUS_OK, k, None


def allocate(mode, s, depth, dist, on_path, is_open, n, params, budget, parent=None, leaf=None):
    """TAE allocation of k_i for every node.

    s: per-node MSVE score (float, fp32 value), depth/dist: geometry,
    on_path: node ∈ Path*, is_open: open block, n: n_i, params: dict with
    alpha gamma lambda_d lambda_delta eta r_min k_min l_tail.
    Returns (status, k: list[int], min_feasible: int|None)."""
    N = len(n)
    n = [int(x) for x in n]
    if mode == MODE_STREAM:
        return stream_targets(parent, leaf, is_open, n, int(params["n_sinks"]), budget)
    # invariant (i): Path* blocks keep k = n (Q19, default) — or, with k_protect > 0,
    # a high floor min(n, k_protect) instead; open blocks are always pinned
    protect = int(params.get("k_protect", 0))
    pinned = [bool(is_open[j]) or (bool(on_path[j]) and protect == 0) for j in range(N)]
    k_min, l_tail, r_min = params["k_min"], params["l_tail"], params["r_min"]

    def pfloor(j, base):
        """Floor of node j: base, raised to min(n, k_protect) on Path* when protected."""
        return max(base, min(n[j], protect)) if (protect and on_path[j]) else base
    size = 2 * N + 2
    E_d = exp_table(params["lambda_d"], size)
    E_D = exp_table(params["lambda_delta"], size)

    def w_of(j):
        return weight(float(s[j]), int(depth[j]), int(dist[j]), not on_path[j],
                      params["gamma"], params["eta"], E_d, E_D)

    k = [n[j] if pinned[j] else 0 for j in range(N)]
    free = [j for j in range(N) if not pinned[j]]
    T = sum(n)
    pinned_total = sum(n[j] for j in range(N) if pinned[j])

    if mode in (MODE_STATIC, MODE_STATIC_DRAIN):
        # Eq. 2: r = clip(α η^{𝟙} s^γ e^{−λ_d d} e^{−λ_Δ Δ}, r_min, 1); Eq. 3 for k
        for j in free:
            r = min(1.0, max(r_min, params["alpha"] * w_of(j)))
            k[j] = pfloor(j, keep_count(r, n[j], k_min, l_tail))
        if mode == MODE_STATIC:
            return STATUS_OK, k, None
        # Alg. 2 Pressure drain: Priority = W_j (Q16), floor K_min (protected
        # Path* blocks: their high floor)
        df = {j: pfloor(j, min(n[j], k_min)) for j in free}
        floor_total = pinned_total + sum(df.values())
        if floor_total > budget:
            return STATUS_INFEASIBLE, None, floor_total
        W = {j: quantize_weight(w_of(j)) for j in free}
        while sum(k) > budget:
            cand = [j for j in free if k[j] > df[j]]
            j = min(cand, key=lambda x: (W[x], -x))
            k[j] = max(df[j], k[j] - 1)
        return STATUS_OK, k, None

    # ---- WATERFILL (optimisation view) ----
    if T <= budget:                                  # step 1: full retention
        return STATUS_OK, list(n), None
    f = {j: pfloor(j, floor_count(n[j], k_min, l_tail, r_min)) for j in free}
    Bp = budget - pinned_total                       # step 4
    if Bp < sum(f.values()):
        return STATUS_INFEASIBLE, None, pinned_total + sum(f.values())
    if Bp >= sum(n[j] for j in free):                # step 5
        for j in free:
            k[j] = n[j]
        return STATUS_OK, k, None
    W = {j: quantize_weight(w_of(j)) for j in free}  # steps 6-7
    P = [j for j in free if W[j] > 0]
    Z = [j for j in free if W[j] == 0]
    if sum(n[j] for j in P) + sum(f[j] for j in Z) <= Bp:   # step 10 saturation
        for j in P:
            k[j] = n[j]
        R = Bp - sum(n[j] for j in P) - sum(f[j] for j in Z)
        kz = proportional_slack([f[j] for j in Z], [n[j] for j in Z], R, Z)
        for j, kk in zip(Z, kz):
            k[j] = kk
        return STATUS_OK, k, None
    for j in Z:
        k[j] = f[j]
    Bpp = Bp - sum(f[j] for j in Z)
    Wl = [W[j] for j in P]
    fl = [f[j] for j in P]
    nl = [n[j] for j in P]
    k_star, active, num, den = box_waterfill(Wl, fl, nl, Bpp)   # step 8
    kp = integerize(Wl, fl, nl, k_star, active, num, den, P)   # step 9
    for j, kk in zip(P, kp):
        k[j] = kk
    return STATUS_OK, k, None


def objective(w, k) -> float:
    """Σ −w_i log k_i, the convex program of P:217-221 (for tests)."""
    return sum(-wi * math.log(ki) for wi, ki in zip(w, k))
