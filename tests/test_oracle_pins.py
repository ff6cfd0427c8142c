"""Pins of the CPU oracle against what the paper and mathematics fix.

Every check here is independent of the oracle's own code path: worked values
quoted from SPEC/SURVEY (tests/golden/spec_vectors.json, each cited), closed
forms, invariants, brute force on tiny inputs, BFS, and library routines
(torch SDPA) on special cases.
"""
import itertools
import json
import math
import os
import random
from fractions import Fraction

import numpy as np
import pytest
import torch

from oracle import attention, geometry, msve, select, tae
from oracle.state import ArborOracle, OracleError, default_params
import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_vectors.json")))


# ---------------------------------------------------------------- geometry
def random_tree(n, rng):
    return [-1] + [int(rng.integers(0, i)) for i in range(1, n)]


def test_geometry_bfs_random_trees():
    """tree_distance equals BFS distances on random trees ≤ 200 nodes."""
    rng = np.random.default_rng(0)
    for n in (1, 2, 7, 50, 200):
        parent = random_tree(n, rng)
        for src in rng.choice(n, size=min(n, 6), replace=False):
            bfs = geometry.bfs_distances(parent, int(src))
            for j in range(n):
                assert geometry.tree_distance(parent, int(src), j) == bfs[j]


def test_geometry_special_cases():
    parent = [-1, 0, 0, 1, 1, 2, 2]        # 3-level binary tree
    assert geometry.depths(parent) == [0, 1, 1, 2, 2, 2, 2]
    assert geometry.tree_distance(parent, 3, 3) == 0
    assert geometry.tree_distance(parent, 1, 3) == 1            # parent↔child
    assert geometry.tree_distance(parent, 3, 4) == 2            # siblings
    assert geometry.tree_distance(parent, 3, 5) == 4            # cousins at depth 2
    assert geometry.root_path(parent, 4) == [0, 1, 4]


def test_geometry_delta_on_path_identity():
    """Δ_i + d_i = d_ℓ* on Path* and Δ = min over several leaves."""
    rng = np.random.default_rng(1)
    for _ in range(20):
        parent = random_tree(60, rng)
        d = geometry.depths(parent)
        leaf = int(rng.integers(60))
        dl = geometry.delta(parent, [leaf])
        for i in geometry.root_path(parent, leaf):
            assert dl[i] + d[i] == d[leaf]
        leaves = [int(x) for x in rng.choice(60, size=3, replace=False)]
        dm = geometry.delta(parent, leaves)
        for i in range(60):
            assert dm[i] == min(geometry.bfs_distances(parent, l)[i] for l in leaves)


# ---------------------------------------------------------------- MSVE
@pytest.mark.parametrize("V", [2, 16, 1024])
def test_uncertainty_extremes(V):
    assert abs(msve.uncertainty([1.0 / V] * V, 0.0, V) - 0.0) < 1e-12   # uniform
    assert abs(msve.uncertainty([1.0], 0.0, V) - 1.0) < 1e-12           # one-hot


def test_uncertainty_bucket_example_and_bound():
    g = GOLD["uncertainty_bucket"]
    assert msve.uncertainty(g["top"], g["other"], g["vocab"]) == g["u"]
    rng = np.random.default_rng(2)
    for _ in range(200):
        V = int(rng.integers(2, 65))
        p = rng.dirichlet(np.ones(V))
        K = int(rng.integers(1, V + 1))
        top = np.sort(p)[::-1][:K]
        exact = msve.uncertainty(list(p), 0.0, V)
        bucket = msve.uncertainty(list(top), float(1 - top.sum()), V)
        assert bucket >= exact - 1e-12          # merging buckets cannot raise H


def test_msve_examples_and_monotonicity():
    g0, g1 = GOLD["msve_theta_zero"], GOLD["msve_example"]
    assert msve.msve_score(g0["theta"], *g0["phi"]) == g0["s"]
    assert abs(msve.msve_score(g1["theta"], *g1["phi"]) - g1["s"]) < 1e-15
    th = (-1.0, 2.0, 1.0, 4.0)
    base = msve.msve_score(th, 0.3, 0.3, 0.3)
    assert msve.msve_score(th, 0.4, 0.3, 0.3) > base
    assert msve.msve_score(th, 0.3, 0.4, 0.3) > base
    assert msve.msve_score(th, 0.3, 0.3, 0.4) > base


def test_attention_feature_closed_forms():
    S = msve.MASS_SCALE
    assert msve.attention_feature(123, 0, 0, 4, 8) == 0.0                 # no queries
    assert msve.attention_feature(4 * 8 * S, 0, 1, 4, 8) == 1.0           # one query, all mass
    assert msve.attention_feature(3 * S, 1 * S, 2, 1, 2) == 0.5
    assert msve.quantize_mass(0.5 / S) == 0 and msve.quantize_mass(1.5 / S) == 2   # half-even


# ---------------------------------------------------------------- TAE
def test_weight_and_keep_count_examples():
    g = GOLD["weight_example"]
    Ed = tae.exp_table(g["lambda_d"], 8)
    ED = tae.exp_table(g["lambda_delta"], 8)
    w = tae.weight(g["s"], g["depth"], g["dist"], False, g["gamma"], 0.8, Ed, ED)
    assert abs(w - g["w"]) <= 2e-17
    for c in GOLD["keep_count"]:
        assert tae.keep_count(c["r"], c["n"], c["k_min"], c["l_tail"]) == c["k"], c
    assert math.floor(0.29 * 100) == 28          # the fp64 pitfall the ε-floor fixes (Q10)


def test_static_monotone_and_offpath_discount():
    """r nondecreasing in s, nonincreasing in Δ; r_off ≤ r_on."""
    Ed, ED = tae.exp_table(0.0, 10), tae.exp_table(0.5, 10)
    r = lambda s, D, off: min(1.0, max(0.05, 0.6 * tae.weight(s, 0, D, off, 1.0, 0.5, Ed, ED)))
    assert r(0.8, 0, True) <= r(0.8, 0, False)
    assert r(0.0, 0, False) == 0.05
    assert r(0.9, 2, False) >= r(0.5, 2, False) >= r(0.5, 3, False)


def test_waterfill_spec_example():
    g = GOLD["waterfill_example"]
    k_star, active, num, den = tae.box_waterfill(g["w"], [0, 0, 0], g["n"], g["budget"])
    assert Fraction(den, num) == Fraction(*g["lambda"])
    assert k_star == [Fraction(*x) for x in g["k_star"]]
    assert tae.integerize(g["w"], [0, 0, 0], g["n"], k_star, active, num, den, [0, 1, 2]) == g["k_int"]


def _kkt_check(W, f, n, B):
    k_star, active, num, den = tae.box_waterfill(W, f, n, B)
    assert sum(k_star) == B
    lam = Fraction(den, num) if num else None
    for j in range(len(W)):
        assert f[j] <= k_star[j] <= n[j]
        if active[j] and lam is None:
            assert k_star[j] == 0                              # λ = ∞: budget = Σ floors
        elif active[j]:
            assert Fraction(W[j]) / k_star[j] == lam          # KKT stationarity
        elif f[j] == n[j]:
            assert k_star[j] == n[j]                           # box of width 0
        elif k_star[j] == n[j] and lam is not None:
            assert Fraction(W[j], n[j]) >= lam                 # capped: w/λ ≥ n
        elif lam is not None:
            assert Fraction(W[j], max(f[j], 1)) <= lam or f[j] == 0
    return k_star


def test_waterfill_kkt_and_scale_invariance_random():
    rng = random.Random(3)
    for _ in range(300):
        m = rng.randint(1, 7)
        n = [rng.randint(1, 40) for _ in range(m)]
        f = [rng.randint(0, x) for x in n]
        W = [rng.randint(1, 10 ** 6) for _ in range(m)]
        if sum(n) <= sum(f):
            continue
        B = rng.randint(sum(f), sum(n) - 1)
        ks = _kkt_check(W, f, n, B)
        c = rng.randint(2, 9)
        ks2, *_ = tae.box_waterfill([w * c for w in W], f, n, B)   # scale invariance
        assert ks2 == ks


def test_integer_rounding_budget_exact_and_near_optimal():
    """Σk = B, f ≤ k ≤ n; brute force on ≤6 nodes, n ≤ 8: the relaxed optimum
    lower-bounds the exhaustive integer optimum, and the rounded allocation is
    within the documented gap."""
    rng = random.Random(4)
    checked = 0
    for _ in range(400):
        m = rng.randint(1, 5)
        n = [rng.randint(1, 8) for _ in range(m)]
        f = [rng.randint(1, x) for x in n]
        W = [rng.randint(1, 50) for _ in range(m)]
        if sum(n) <= sum(f):
            continue
        B = rng.randint(sum(f), sum(n) - 1)
        ks, active, num, den = tae.box_waterfill(W, f, n, B)
        k = tae.integerize(W, f, n, ks, active, num, den, list(range(m)))
        assert sum(k) == B and all(f[j] <= k[j] <= n[j] for j in range(m))
        best = min(tae.objective(W, c) for c in itertools.product(*[range(f[j], n[j] + 1) for j in range(m)])
                   if sum(c) == B)
        relaxed = tae.objective(W, [float(x) for x in ks])
        assert relaxed <= best + 1e-9
        gap = sum(W[j] * math.log(1 + 1 / max(1, math.floor(ks[j]))) for j in range(m) if active[j])
        assert tae.objective(W, k) - best <= gap + 1e-9
        checked += 1
    assert checked > 200


def _c1_inputs():
    g = GOLD["c1_waterfill"]
    p = dict(default_params(), **g["params"])
    parent = g["parent"]
    d = geometry.depths(parent)
    dist = geometry.delta(parent, g["active"])
    ps = geometry.path_star(parent, g["active"])
    on = [i in ps for i in range(7)]
    return g, p, d, dist, on


def test_c1_worked_answer():
    g, p, d, dist, on = _c1_inputs()
    for j, D in g["dist_offpath"].items():
        assert dist[int(j)] == D
    Ed, ED = tae.exp_table(p["lambda_d"], 16), tae.exp_table(p["lambda_delta"], 16)
    for j, Wj in g["W_offpath"].items():
        j = int(j)
        w = tae.weight(1.0, d[j], dist[j], True, p["gamma"], p["eta"], Ed, ED)
        assert tae.quantize_weight(w) == Wj
    st, k, _ = tae.allocate(tae.MODE_WATERFILL, [1.0] * 7, d, dist, on, [0] * 7, g["n"], p,
                            g["budget"])
    assert st == 0 and k == g["k"] and sum(k) == g["budget"]


def test_allocate_invariants_random():
    """Pinned k = n; Σk = B when T > B and feasible; floors hold; B ≥ T → k = n;
    identical off-path nodes get equal k; infeasible reports min feasible."""
    rng = np.random.default_rng(5)
    p = default_params()
    for trial in range(150):
        N = int(rng.integers(2, 40))
        parent = random_tree(N, rng)
        n = [int(x) for x in rng.integers(1, 64, size=N)]
        active = [int(x) for x in rng.choice(N, size=int(rng.integers(1, min(N, 3) + 1)), replace=False)]
        is_open = [0] * N
        d = geometry.depths(parent)
        dist = geometry.delta(parent, active)
        ps = geometry.path_star(parent, active)
        on = [i in ps for i in range(N)]
        s = [float(np.float32(x)) for x in rng.random(N)]
        T = sum(n)
        B = int(rng.integers(0, T + 20))
        st, k, mf = tae.allocate(tae.MODE_WATERFILL, s, d, dist, on, is_open, n, p, B)
        floors = [tae.floor_count(n[j], p["k_min"], p["l_tail"], p["r_min"]) for j in range(N)]
        need = sum(n[j] if on[j] else floors[j] for j in range(N))
        if need > B:
            assert st == tae.STATUS_INFEASIBLE and mf == need
            continue
        assert st == 0
        for j in range(N):
            assert (k[j] == n[j]) if on[j] else (floors[j] <= k[j] <= n[j])
        assert sum(k) == min(B, T)
        if B >= T:
            assert k == n
    # symmetry: two identical off-path siblings
    parent = [-1, 0, 0, 0]
    n = [10, 20, 20, 20]
    d = geometry.depths(parent)
    dist = geometry.delta(parent, [1])
    on = [True, True, False, False]
    st, k, _ = tae.allocate(tae.MODE_WATERFILL, [0.5, 0.5, 0.7, 0.7], d, dist, on, [0] * 4, n, p, 48)
    assert k[2] == k[3] and sum(k) == 48


def test_ablation_variants_msve_only_and_tae_only():
    """P:408-414 ablations as parameter settings of the same allocation.
    MSVE-only (λ_d = λ_Δ = 0, η = 1): the weight is s^γ alone, so on random trees two
    non-pinned nodes with equal (s, n) get k within 1 of each other and a larger s never gets
    a smaller k at equal n.  TAE-only (s ≡ const): k follows the tree alone — equal (Δ, n) off
    the path (depth unused at λ_d = 0, η = 1) → k within 1, larger Δ → k no larger."""
    rng = np.random.default_rng(41)
    for trial in range(120):
        N = int(rng.integers(6, 40))
        parent = random_tree(N, rng)
        leaves = [i for i in range(N) if i not in set(parent)]
        active = [int(rng.choice(leaves))]
        d = geometry.depths(parent)
        dist = geometry.delta(parent, active)
        ps = geometry.path_star(parent, active)
        on = [i in ps for i in range(N)]
        n = [int(x) for x in rng.choice([24, 48], size=N)]
        free = [j for j in range(N) if not on[j]]
        B = sum(n[j] for j in range(N) if on[j]) + sum(n[j] for j in free) // 3
        if trial % 2 == 0:      # MSVE-only
            p = default_params(lambda_d=0.0, lambda_delta=0.0, eta=1.0, r_min=0.0)
            s = [float(np.float32(x)) for x in rng.choice([0.2, 0.5, 0.9], size=N)]
            key = lambda j: (s[j], n[j])                       # noqa: E731
            order = lambda j: s[j]                             # noqa: E731
            sign = 1
        else:                   # TAE-only
            p = default_params(lambda_d=0.0, lambda_delta=0.7, eta=1.0, r_min=0.0)
            s = [0.5] * N
            key = lambda j: (dist[j], n[j])                    # noqa: E731
            order = lambda j: dist[j]                          # noqa: E731
            sign = -1
        st, k, _ = tae.allocate(tae.MODE_WATERFILL, s, d, dist, on, [0] * N, n, p, B)
        assert st == 0 and sum(k) == B
        for a in free:
            for b in free:
                if key(a) == key(b):
                    assert abs(k[a] - k[b]) <= 1, (trial, a, b, k[a], k[b])
                elif n[a] == n[b] and sign * (order(a) - order(b)) > 0:
                    assert k[a] >= k[b], (trial, a, b, k[a], k[b])


def test_allocate_zero_weights_saturation():
    """W rounding to 0 (s ≈ 0): floor only unless positive-weight nodes saturate;
    then the remainder is spread over zero-weight nodes by slack (§8(c).1 step 10)."""
    p = default_params(k_min=2, l_tail=2, r_min=0.0)
    parent = [-1, 0, 0, 0]
    d, dist = geometry.depths(parent), geometry.delta(parent, [0])
    on = [True, False, False, False]
    n = [4, 10, 10, 10]
    st, k, _ = tae.allocate(tae.MODE_WATERFILL, [1.0, 0.9, 0.0, 0.0], d, dist, on, [0] * 4, n, p, 4 + 10 + 2 + 2)
    assert k == [4, 10, 2, 2]
    st, k, _ = tae.allocate(tae.MODE_WATERFILL, [1.0, 0.9, 0.0, 0.0], d, dist, on, [0] * 4, n, p, 4 + 10 + 9)
    assert k == [4, 10, 5, 4] and sum(k) == 23


def test_static_drain_matches_unit_step():
    """STATIC_DRAIN = Alg. 2 P:579-583 unit-step drain; chunked form equal."""
    rng = np.random.default_rng(6)
    p = default_params(alpha=3.0)
    for _ in range(60):
        N = int(rng.integers(2, 25))
        parent = random_tree(N, rng)
        n = [int(x) for x in rng.integers(1, 40, size=N)]
        d = geometry.depths(parent)
        dist = geometry.delta(parent, [N - 1])
        ps = geometry.path_star(parent, [N - 1])
        on = [i in ps for i in range(N)]
        s = [float(np.float32(x)) for x in rng.random(N)]
        st0, k0, _ = tae.allocate(tae.MODE_STATIC, s, d, dist, on, [0] * N, n, p, 0)
        B = int(rng.integers(sum(min(n[j], p["k_min"]) if not on[j] else n[j] for j in range(N)), sum(k0) + 1))
        st, k, _ = tae.allocate(tae.MODE_STATIC_DRAIN, s, d, dist, on, [0] * N, n, p, B)
        assert st == 0 and sum(k) == min(B, sum(k0)) if sum(k0) > B else k == k0
        # chunked drain: walk priority order once
        Ed, ED = tae.exp_table(p["lambda_d"], 2 * N + 2), tae.exp_table(p["lambda_delta"], 2 * N + 2)
        W = {j: tae.quantize_weight(tae.weight(s[j], d[j], dist[j], not on[j], p["gamma"], p["eta"], Ed, ED))
             for j in range(N) if not on[j]}
        kc = list(k0)
        excess = sum(kc) - B
        for j in sorted(W, key=lambda x: (W[x], -x)):
            if excess <= 0:
                break
            dd = min(excess, max(0, kc[j] - p["k_min"]))
            kc[j] -= dd
            excess -= dd
        assert kc == k


# ---------------------------------------------------------------- selection
def test_select_spec_example():
    g = GOLD["select_example"]
    R = select.retained_set(list(range(g["n"])), g["n"], g["k"], g["l_tail"], np.array(g["A"], np.float32))
    assert R == g["kept"]


def test_select_properties_random():
    """|ℛ| = k, tail ⊆ ℛ, ℛ ⊆ C, every kept heavy hitter outranks every dropped
    candidate (defining property of top-m), k ≤ L_tail → last k, k = n → all."""
    rng = np.random.default_rng(7)
    for _ in range(500):
        n = int(rng.integers(1, 40))
        lt = int(rng.integers(0, 10))
        A = rng.integers(0, 5, size=n).astype(np.float32) * np.float32(0.25)   # many exact ties
        kept = list(range(n))
        k1 = int(rng.integers(0, n + 1))
        R = select.retained_set(kept, n, k1, lt, A)
        assert len(R) == k1 and set(R) <= set(kept)
        tl = min(lt, n)
        if k1 <= tl:
            assert R == list(range(n - k1, n))
        else:
            assert set(range(n - tl, n)) <= set(R)
            dropped = [t for t in kept if t not in R]
            heavy = [t for t in R if t < n - tl]
            for x in heavy:
                for y in dropped:
                    assert (A[x], x) > (A[y], y)
        if k1 == n:
            assert R == kept
        # a second eviction never grows and only picks from the survivors (Q2)
        k2 = int(rng.integers(0, k1 + 1))
        R2 = select.retained_set(R, n, k2, lt, A)
        assert set(R2) <= set(R) and len(R2) == k2


def test_trim_prefix_equivalence():
    """retained_set equals SPEC S:402's trim prefix oracle over tail ∪ all candidates."""
    rng = np.random.default_rng(8)
    for _ in range(300):
        n = int(rng.integers(1, 30))
        lt = int(rng.integers(1, 8))
        A = rng.random(n).astype(np.float32)
        k = int(rng.integers(min(lt, n), n + 1))
        tail = list(range(n - min(lt, n), n))
        cand = [t for t in range(n) if t not in tail]
        assert select.retained_set(list(range(n)), n, k, lt, A) == select.trim_prefix(tail, cand, k, A)


def test_select_rejects_invalid_scores():
    with pytest.raises(ValueError):
        select.f32_bits(-1.0)
    with pytest.raises(ValueError):
        select.f32_bits(float("nan"))
    assert select.f32_bits(-0.0) == 0


# ---------------------------------------------------------------- attention
def test_attention_matches_torch_sdpa_full_retention():
    """Full retention + one leaf = standard decode attention over the
    concatenated path (torch SDPA, fp64)."""
    rng = np.random.default_rng(9)
    for T, G in ((1, 1), (37, 4), (300, 8)):
        q = rng.standard_normal((G, 64))
        K = rng.standard_normal((T, 64))
        V = rng.standard_normal((T, 64))
        o, lse, p = attention.attend(q, K, V)
        ref = torch.nn.functional.scaled_dot_product_attention(
            torch.tensor(q)[None, :, None, :], torch.tensor(K)[None, None].expand(1, G, T, 64),
            torch.tensor(V)[None, None].expand(1, G, T, 64))[0, :, 0, :].numpy()
        assert np.allclose(o, ref, rtol=1e-12, atol=1e-12)
        z = torch.tensor(q) @ torch.tensor(K).T / 8.0
        assert np.allclose(lse, torch.logsumexp(z, dim=1).numpy(), rtol=1e-12)
        assert np.allclose(p.sum(axis=1), 1.0)


def test_attention_closed_forms():
    rng = np.random.default_rng(10)
    v = rng.standard_normal((1, 16))
    o, lse, _ = attention.attend(rng.standard_normal((2, 16)), rng.standard_normal((1, 16)), v)
    assert np.allclose(o, v)                               # single visible token → o = v
    K = np.tile(rng.standard_normal((1, 16)), (9, 1))
    V = rng.standard_normal((9, 16))
    o, lse, p = attention.attend(rng.standard_normal((3, 16)), K, V)
    assert np.allclose(o, V.mean(axis=0)[None])            # identical keys → mean(V)
    q0 = np.zeros((2, 16))
    o, lse, p = attention.attend(q0, rng.standard_normal((7, 16)), rng.standard_normal((7, 16)))
    assert np.allclose(p, 1.0 / 7) and np.allclose(lse, math.log(7))   # q = 0 → uniform


# ---------------------------------------------------------------- state machine
def _small_state(levels=3, width=2, t_node=12, L=2, H=2, G=2, d=16, P=4, seed=0, params=None):
    tree = synth.full_tree(levels, width, t_node, seed)
    T = tree.total_tokens
    K, V, E = synth.make_kv(L, H, T, d, "f32", seed, tree.span_start, tree.span_len)
    params = params or default_params(k_min=2, l_tail=3, r_min=0.0)
    pages = sum(-(-int(x) // P) for x in tree.span_len) + 8
    o = ArborOracle(K.double().numpy(), V.double().numpy(), H * G, P, pages, params)
    for i in range(tree.num_nodes):
        o.open_node(i, int(tree.span_start[i]))
        o.append(i, int(tree.span_len[i]))
        o.close_node(i)
    return tree, o, E


def test_state_pages_conserved_and_evict_rehydrate_roundtrip():
    tree, o, E = _small_state()
    tree.active = [synth.leaves_of(tree)[0]]
    q = synth.make_queries(1, o.L, o.Hq, o.d, "f32", 1, E).double().numpy()
    for _ in range(3):
        o.score_accumulate(tree, q)
    a, s = o.msve(tree)
    assert all(0.0 <= x <= 1.0 for x in a)
    full = [o.kept[i].copy() for i in range(tree.num_nodes)]
    B = tree.total_tokens * 3 // 4
    k = o.allocate(tree, s, B)
    assert sum(k) == B
    o.evict(tree, k)
    for i in range(tree.num_nodes):
        assert o.k_cur(i) == k[i]
    assert sum(len(pg) for pg in o.pages) + len(o.free) == o.num_pages
    # backtrack: make another leaf active and rehydrate its path (Alg. 2)
    other = synth.leaves_of(tree)[-1]
    tree.active = [other]
    path = geometry.root_path(tree.parent, other)
    need = [i for i in path if o.k_cur(i) < o.n[i]]
    assert o.rehydrate(path) == len(need) and o.rehydrations == len(need)
    for i in path:
        assert np.array_equal(o.kept[i], full[i])         # bit-exact restore of the set
    assert o.rehydrate(path) == 0                          # full nodes: no-op, not counted
    assert sum(len(pg) for pg in o.pages) + len(o.free) == o.num_pages


def test_rehydrate_slot_layout_worked_example():
    """DESIGN.md Q23r, worked by hand: P = 4, a 10-token block (pages p0 p1 p2 for slots
    0-3, 4-7, 8-11) evicted to k = 3: its window is the last 3 slots 7, 8, 9 holding
    positions [7, 2, 9] — page p0 freed, koff = 3 in the live list [p1, p2].  Rehydration
    pops one page (the top of the LIFO free stack) for the freed slots 0-3 and puts every
    position back in its slot."""
    tree = synth.full_tree(1, 1, 10)
    K = np.zeros((1, 1, tree.total_tokens, 2))
    o = ArborOracle(K, K, 1, 4, 16, default_params())
    o.open_node(0, 0)
    o.append(0, 10)
    o.close_node(0)
    p0, p1, p2 = o.pages[0]
    o.free.append(p0)                          # the evicted state by construction
    o.pages[0] = [p1, p2]
    o.koff[0] = 3
    o.kept[0] = np.array([[[7, 2, 9]]], dtype=np.int64)
    stack = list(o.free)
    assert o.rehydrate([0]) == 1
    assert o.kept[0].tolist() == [[list(range(10))]]
    assert o.koff[0] == 0
    assert o.pages[0] == [stack[-1], p1, p2] and stack[-1] == p0
    assert o.free == stack[:-1]


def test_state_unlimited_budget_is_full_retention():
    tree, o, E = _small_state(seed=3)
    tree.active = [synth.leaves_of(tree)[1]]
    q = synth.make_queries(1, o.L, o.Hq, o.d, "f32", 2, E).double().numpy()
    o_full, _ = o.decode(tree, q)
    o.score_accumulate(tree, q)
    a, s = o.msve(tree)
    k = o.allocate(tree, s, 10 ** 9)
    assert k == o.n
    assert o.evict(tree, k) == 0
    o2, _ = o.decode(tree, q)
    assert np.array_equal(o2, o_full)


def test_state_score_mass_conservation():
    """Per decode step each row's ΣΔA = n_A·G."""
    tree, o, E = _small_state(levels=3, width=3, seed=4)
    tree.active = synth.leaves_of(tree)[:3]
    q = synth.make_queries(3, o.L, o.Hq, o.d, "f32", 3, E).double().numpy()
    before = o.A.sum(axis=2)
    o.score_accumulate(tree, q)
    assert np.allclose(o.A.sum(axis=2) - before, 3 * o.G, rtol=1e-12)


def test_state_lifecycle_errors():
    tree, o, E = _small_state()
    with pytest.raises(OracleError):
        o.close_node(0)
    o.open_node(tree.num_nodes, tree.end_position())
    with pytest.raises(OracleError):
        o.rehydrate([tree.num_nodes])


def test_state_hole_filling_layout():
    """DESIGN.md Q23* (end-window hole filling): after eviction every row holds exactly the
    retained set; the new block is the last k_app of the old valid slots (w = k_cur − k_app
    onward); retained rows already inside the window keep their slot; the holes there are
    filled, in ascending order, by the retained rows from slots < w in ascending order.  The
    page list loses its ⌊(koff + w)/P⌋ leading pages (pushed descending), koff ← (koff + w)
    mod P, and the live list is exactly ⌈(koff + k_cur)/P⌉ pages — checked over two rounds
    of eviction, so a block that already has koff > 0 is evicted again."""
    tree, o, E = _small_state(levels=3, width=3, t_node=20, seed=6)
    tree.active = [synth.leaves_of(tree)[0]]
    q = synth.make_queries(1, o.L, o.Hq, o.d, "f32", 9, E).double().numpy()
    for frac in (0.6, 0.35):
        for _ in range(4):
            o.score_accumulate(tree, q)
        before = [o.kept[i].copy() for i in range(tree.num_nodes)]
        pages_before = [list(o.pages[i]) for i in range(tree.num_nodes)]
        koff_before = list(o.koff)
        free_before = list(o.free)
        a, s = o.msve(tree)
        k = o.allocate(tree, s, int(tree.total_tokens * frac))
        o.evict(tree, k)
        Af = o.A.astype(np.float32)
        pushed = []
        for i in range(tree.num_nodes):
            kc0 = before[i].shape[-1]
            assert 0 <= o.koff[i] < o.P
            assert len(o.pages[i]) == -(-(o.koff[i] + o.k_cur(i)) // o.P)
            if o.k_cur(i) == kc0:
                assert o.pages[i] == pages_before[i] and o.koff[i] == koff_before[i]
                continue
            ka, a0, n = o.k_cur(i), o.span_start[i], o.n[i]
            w = kc0 - ka
            c = koff_before[i] + w
            drop = c // o.P if ka else len(pages_before[i])
            assert o.pages[i] == pages_before[i][drop:]
            assert o.koff[i] == (c % o.P if ka else 0)
            pushed += list(reversed(pages_before[i][:drop]))
            for l in range(o.L):
                for h in range(o.H):
                    old = [int(x) for x in before[i][l, h]]
                    new = [int(x) for x in o.kept[i][l, h]]
                    R = select.retained_set(old, n, ka, o.params["l_tail"], Af[l, h, a0:a0 + n])
                    assert sorted(new) == R
                    stay = [s_ for s_ in range(w, kc0) if old[s_] in R]
                    assert all(new[s_ - w] == old[s_] for s_ in stay)
                    holes = [s_ for s_ in range(w, kc0) if old[s_] not in R]
                    movers = [old[s_] for s_ in range(w) if old[s_] in R]
                    assert [new[s_ - w] for s_ in holes] == movers
        assert o.free == free_before + pushed


# ---------------------------------------------------------------- f4 intra-block variants
@pytest.mark.parametrize("n,k,l_tail,s", [(40, 13, 4, 3), (17, 9, 2, 4), (64, 20, 8, 0), (12, 5, 5, 2)])
def test_select_variants_closed_forms(n, k, l_tail, s):
    """Tail-only and Sinks + Tail from full retention reduce to intervals:
    Tail keeps the last k positions; Sinks + Tail keeps the global sinks — the first
    min(s, m) positions of the ROOT block (the initial prompt; m = k − |tail|) —
    and the most recent k − min(s, m); in any other block it is Tail-only.  HEAVY keeps the
    root's sinks before any heavy hitter.  None of the recency rules depends on A."""
    rng = np.random.default_rng(n * 7 + k)
    A = rng.random(n).astype(np.float32)
    full = list(range(n))
    tl = min(l_tail, n)
    last = list(range(n - k, n))
    assert select.retained_set(full, n, k, l_tail, A, select.TAIL) == last
    assert select.retained_set(full, n, k, l_tail, A, select.TAIL, s, is_root=True) == last
    assert select.retained_set(full, n, k, l_tail, A, select.SINKS_TAIL, s) == last
    m = max(k - tl, 0)
    sk = min(s, m) if k > tl else 0
    want = sorted(set(range(sk)) | set(range(n - (k - sk), n)))
    assert select.retained_set(full, n, k, l_tail, A, select.SINKS_TAIL, s, is_root=True) == want
    # HEAVY in the root: the sinks, then the top-(m − sinks) of the rest by A, plus the tail
    hv = select.retained_set(full, n, k, l_tail, A, select.HEAVY, s, is_root=True)
    rest = sorted(range(sk, n - tl), key=lambda t: (A[t], t), reverse=True)[:m - sk]
    assert hv == sorted(set(range(sk)) | set(rest) | set(range(n - tl, n)))
    A2 = rng.permutation(A)
    for mode in (select.TAIL, select.SINKS_TAIL):
        assert (select.retained_set(full, n, k, l_tail, A, mode, s, is_root=True) ==
                select.retained_set(full, n, k, l_tail, A2, mode, s, is_root=True))


def test_select_variants_compose():
    """Evicting to k1 then k2 < k1 equals evicting to k2 directly (the rules rank the same
    positions the same way at every step)."""
    rng = np.random.default_rng(3)
    for mode in (select.HEAVY, select.TAIL, select.SINKS_TAIL):
        for _ in range(20):
            n = int(rng.integers(8, 60))
            A = rng.random(n).astype(np.float32)
            k1 = int(rng.integers(1, n + 1))
            k2 = int(rng.integers(0, k1 + 1))
            r1 = select.retained_set(list(range(n)), n, k1, 3, A, mode, 2)
            assert (select.retained_set(r1, n, k2, 3, A, mode, 2) ==
                    select.retained_set(list(range(n)), n, k2, 3, A, mode, 2))


def test_no_rehydrate_is_irreversible():
    """with rehydration disabled an evicted block never comes back."""
    tree, orc, _ = _small_state(params=default_params(k_min=2, l_tail=3, r_min=0.0,
                                                       no_rehydrate=True))
    tree.active = [synth.leaves_of(tree)[0]]
    N = len(orc.n)
    k = [2] * N
    orc.evict(tree, k)
    before = [orc.k_cur(i) for i in range(N)]
    assert orc.rehydrate(list(range(N))) == 0
    assert [orc.k_cur(i) for i in range(N)] == before


# ---------------------------------------------------------------- round 2: path assembly, A_i(t)
def _root_chain(parent, leaf):
    """Root→leaf chain by a plain parent walk (independent of oracle.geometry)."""
    out = []
    x = int(leaf)
    while x >= 0:
        out.append(x)
        x = int(parent[x])
    return out[::-1]


def _path_kv(o, tree, leaf, l, h):
    """Visible positions of (leaf, l, h): every node of the root chain, its kept positions
    sorted ascending — assembled here without oracle.attention."""
    pos = []
    for i in _root_chain(tree.parent, leaf):
        pos.extend(sorted(int(tree.span_start[i]) + int(t) for t in o.kept[i][l, h]))
    return np.array(pos, dtype=np.int64)


def _sdpa(q, K, V):
    """torch SDPA (fp64, CPU) for G query rows over one KV sequence, and its logsumexp."""
    G, d = q.shape
    T = K.shape[0]
    qt, Kt, Vt = torch.tensor(q), torch.tensor(K), torch.tensor(V)
    o = torch.nn.functional.scaled_dot_product_attention(
        qt[None, :, None, :], Kt[None, None].expand(1, G, T, d),
        Vt[None, None].expand(1, G, T, d))[0, :, 0, :]
    z = qt @ Kt.T / math.sqrt(d)
    return o.numpy(), torch.logsumexp(z, dim=1).numpy(), torch.softmax(z, dim=1).numpy()


@pytest.mark.parametrize("evict", [False, True])
def test_state_decode_is_sdpa_over_concatenated_path(evict):
    """Tree decode attention of every active leaf = torch SDPA over the concatenation of its
    root→leaf chain's retained K/V (full retention: standard causal decode over the path
    sequence); after an eviction, over the kept positions."""
    tree, o, E = _small_state(levels=3, width=3, t_node=10, seed=11)
    leaves = synth.leaves_of(tree)
    tree.active = [leaves[0]]
    q1 = synth.make_queries(1, o.L, o.Hq, o.d, "f32", 5, E).double().numpy()
    o.score_accumulate(tree, q1)
    if evict:
        a, s = o.msve(tree)
        o.evict(tree, o.allocate(tree, s, tree.total_tokens // 2))
    tree.active = [leaves[0], leaves[4], leaves[-1]]
    q = synth.make_queries(3, o.L, o.Hq, o.d, "f32", 6, E).double().numpy()
    out, lse = o.decode(tree, q)
    for b, leaf in enumerate(tree.active):
        for l in range(o.L):
            for h in range(o.H):
                pos = _path_kv(o, tree, leaf, l, h)
                gs = slice(h * o.G, (h + 1) * o.G)
                ref_o, ref_l, _ = _sdpa(q[b, l, gs], o.K[l, h, pos], o.V[l, h, pos])
                assert np.allclose(out[b, l, gs], ref_o, rtol=1e-12, atol=1e-12)
                assert np.allclose(lse[b, l, gs], ref_l, rtol=1e-12, atol=1e-12)


def test_state_multi_leaf_equals_single_leaf_runs():
    """Tree sharing changes nothing: an n_A-leaf decode equals n_A
    single-leaf decodes, and the n_A-leaf score pass adds exactly the sum of the single-leaf
    passes' attention mass (A is additive over queries)."""
    tree, o, E = _small_state(levels=3, width=3, t_node=9, seed=12)
    leaves = synth.leaves_of(tree)
    act = [leaves[1], leaves[2], leaves[7]]
    q = synth.make_queries(3, o.L, o.Hq, o.d, "f32", 7, E).double().numpy()
    tree.active = act
    out, lse = o.decode(tree, q)
    A0 = o.A.copy()
    o.score_accumulate(tree, q, lse)
    dA_multi = o.A - A0
    o.A[:] = A0
    for b, leaf in enumerate(act):
        tree.active = [leaf]
        ob, lb = o.decode(tree, q[b:b + 1])
        assert np.array_equal(ob[0], out[b]) and np.array_equal(lb[0], lse[b])
        o.score_accumulate(tree, q[b:b + 1], lb)
    assert np.allclose(o.A - A0, dA_multi, rtol=1e-13, atol=1e-15)


def test_accumulated_attention_counts_later_queries_only():
    """A_i(t) = Σ_{u>b_i} Σ_{l,h} Attn_{u→t}: queries of an open block (the block
    they belong to, Q25) add nothing to that block's own tokens while it is open; after it
    closes, only queries of later blocks count.  The reference A is rebuilt here from torch
    softmax weights over the independently assembled path."""
    tree, o, E = _small_state(levels=2, width=2, t_node=6, L=1, H=2, G=2, d=16, P=4, seed=13)
    gen = torch.Generator().manual_seed(5)
    A_ref = np.zeros_like(o.A)
    K, V = o.K, o.V

    def decode_from(leaf, step, own_open):
        q = synth.make_queries(1, o.L, o.Hq, o.d, "f32", step, E).double().numpy()
        tree.active = [leaf]
        o.score_accumulate(tree, q)
        for l in range(o.L):
            for h in range(o.H):
                pos = _path_kv(o, tree, leaf, l, h)
                _, _, p = _sdpa(q[0, l, h * o.G:(h + 1) * o.G], K[l, h, pos], V[l, h, pos])
                w = p.sum(axis=0)
                if own_open:
                    a0, n = int(tree.span_start[leaf]), int(tree.span_len[leaf])
                    w = np.where((pos >= a0) & (pos < a0 + n), 0.0, w)
                A_ref[l, h, pos] += w

    # a closed active leaf: its query is the next token (u > b_ℓ), so ℓ's tokens count
    decode_from(1, 100, own_open=False)
    # grow an open child c under leaf 2, one token per step; c's tokens never gain mass
    c = tree.add_node(2, tree.end_position(), 0, True, 0.5, 0.5)
    o.open_node(c, int(tree.span_start[c]))
    T_extra = 5
    o.K = np.concatenate([K, torch.randn(o.L, o.H, T_extra, o.d, generator=gen, dtype=torch.float64).numpy()], axis=2)
    o.V = np.concatenate([V, torch.randn(o.L, o.H, T_extra, o.d, generator=gen, dtype=torch.float64).numpy()], axis=2)
    o.A = np.concatenate([o.A, np.zeros((o.L, o.H, T_extra))], axis=2)
    A_ref = np.concatenate([A_ref, np.zeros((o.L, o.H, T_extra))], axis=2)
    K, V = o.K, o.V
    for step in range(3):
        o.append(c, 1)
        tree.span_len[c] += 1
        decode_from(c, 200 + step, own_open=True)
        a0 = int(tree.span_start[c])
        assert not o.A[:, :, a0:a0 + int(tree.span_len[c])].any()
    # close c: Mclose_c is 0 (no mass while open); a grandchild g's queries now count for c
    o.close_node(c)
    tree.is_open[c] = 0
    assert o.Mclose[c] == 0 and o.Nq[c] == 0
    g = tree.add_node(c, tree.end_position(), 0, True, 0.5, 0.5)
    o.open_node(g, int(tree.span_start[g]))
    for step in range(2):
        o.append(g, 1)
        tree.span_len[g] += 1
        decode_from(g, 300 + step, own_open=True)
    assert np.allclose(o.A, A_ref, rtol=1e-12, atol=1e-15)
    a0 = int(tree.span_start[c])
    assert o.A[:, :, a0:a0 + int(tree.span_len[c])].sum() > 0
    assert o.Nq[c] == 2
    # its feature is exactly the post-close mass per query row (Q4)
    a, _ = o.msve(tree)
    m = sum(round(math.fsum(A_ref[l, h, a0:a0 + int(tree.span_len[c])]) * 2 ** 24)
            for l in range(o.L) for h in range(o.H))
    assert abs(a[c] - m / 2 ** 24 / (2 * o.L * o.Hq)) < 1e-12


def test_node_mass_counts_frozen_evicted_scores():
    """m_{l,h,i} sums the whole span, kept and evicted positions alike; evicted A is frozen
    (SPEC S:429): eviction leaves every node mass unchanged, later score passes never
    touch evicted positions, and Mass_i = Σ_rows round(2^24·Σ_span A) (reference sums with
    math.fsum: each row may differ from the fp64 running sum by at most one unit)."""
    tree, o, E = _small_state(levels=3, width=2, t_node=16, seed=14)
    leaves = synth.leaves_of(tree)
    tree.active = [leaves[0]]
    for st in range(3):
        o.score_accumulate(tree, synth.make_queries(1, o.L, o.Hq, o.d, "f32", 40 + st, E).double().numpy())
    before = o.masses()
    a, s = o.msve(tree)
    o.evict(tree, o.allocate(tree, s, tree.total_tokens * 3 // 5))
    assert o.masses() == before
    evicted = np.ones_like(o.A, dtype=bool)
    for i in range(tree.num_nodes):
        for l in range(o.L):
            for h in range(o.H):
                evicted[l, h, int(tree.span_start[i]) + o.kept[i][l, h]] = False
    assert evicted.any()
    A_ev = o.A[evicted].copy()
    tree.active = [leaves[-1]]
    o.score_accumulate(tree, synth.make_queries(1, o.L, o.Hq, o.d, "f32", 50, E).double().numpy())
    assert np.array_equal(o.A[evicted], A_ev)
    for i in range(tree.num_nodes):
        a0, n = int(tree.span_start[i]), int(tree.span_len[i])
        ref = sum(round(math.fsum(o.A[l, h, a0:a0 + n]) * 2 ** 24) for l in range(o.L) for h in range(o.H))
        assert abs(o.masses()[i] - ref) <= o.L * o.H


@pytest.mark.parametrize("name", ["hole_fill_example", "hole_fill_example2"])
def test_hole_fill_worked_example(name):
    """Q23* slot order and page accounting on the hand-worked examples of tests/golden (the
    first from SPEC S:392; the second with a staying row between two holes)."""
    g = GOLD[name]
    A_row = GOLD["select_example"]["A"] if name == "hole_fill_example" else g["A"]
    tree = synth.SynthTree(np.array([-1, 0], np.int32), np.array([0, 10], np.int64),
                           np.array([10, 4], np.int32), np.zeros(2, np.uint8),
                           np.zeros(2, np.float32), np.zeros(2, np.float32), [1])
    L, H, d = 1, 1, 4
    K = np.zeros((L, H, 14, d))
    o = ArborOracle(K, K, 1, g["page_size"], 8, default_params(k_min=1, l_tail=3, r_min=0.0, n_sinks=0))
    for i in range(2):
        o.open_node(i, int(tree.span_start[i]))
        o.append(i, int(tree.span_len[i]))
        o.close_node(i)
    tree.active = [1]
    A = np.zeros((L, H, 14), np.float32)
    A[0, 0, :10] = A_row
    pages0 = list(o.pages[0])
    # the root is on Path*: evict node 0 through a tree in which node 1 hangs off elsewhere
    tree2 = synth.SynthTree(np.array([-1, -1], np.int32), tree.span_start, tree.span_len,
                            tree.is_open, tree.v, tree.u, [1])
    o.evict(tree2, [g["k_app"], 4], A_f32=A)
    assert sorted(o.kept[0][0, 0].tolist()) == g["retained"]
    assert o.kept[0][0, 0].tolist() == g["new_slots"]
    assert o.koff[0] == g["koff"]
    assert o.pages[0] == pages0[g["freed_pages_front"]:]
    assert o.free[-g["freed_pages_front"]:] == list(reversed(pages0[:g["freed_pages_front"]]))


def test_k_protect_reduces_to_pinning_and_keeps_floors():
    """P:104 "k_i = n_i or a high floor k_protect": a floor at least every n is the pinned
    policy exactly (all modes); a lower floor keeps every Path* block at ≥ min(n, k_protect),
    still meets the budget exactly (WATERFILL) and reports min_feasible with those floors."""
    rng = np.random.default_rng(77)
    for trial in range(200):
        N = int(rng.integers(2, 25))
        parent = [-1] + [int(rng.integers(0, i)) for i in range(1, N)]
        n = [int(x) for x in rng.integers(1, 20, size=N)]
        kids = set(parent[1:])
        leaves = [i for i in range(N) if i not in kids]
        act = sorted(set(int(x) for x in rng.choice(leaves, size=min(2, len(leaves)), replace=False)))
        d = geometry.depths(parent)
        dist = geometry.delta(parent, act)
        on = [i in geometry.path_star(parent, act) for i in range(N)]
        opn = [False] * N
        s = [float(np.float32(x)) for x in rng.random(N)]
        B = int(rng.integers(sum(n) // 4, sum(n)))
        for mode in (0, 1, 2):
            base = default_params(k_min=int(rng.integers(0, 4)), l_tail=int(rng.integers(0, 4)))
            ref = tae.allocate(mode, s, d, dist, on, opn, n, base, B)
            big = tae.allocate(mode, s, d, dist, on, opn, n, dict(base, k_protect=max(n)), B)
            assert ref == big, (trial, mode)
            prot = int(rng.integers(1, 10))
            st, k, mf = tae.allocate(mode, s, d, dist, on, opn, n, dict(base, k_protect=prot), B)
            if st != 0:
                continue
            for j in range(N):
                if on[j]:
                    assert k[j] >= min(n[j], prot)
            if mode == 0 and sum(n) > B:
                assert sum(k) == B


def test_thin_slice_rows_and_shared_selection_reduce_to_per_row():
    """Slice rows = the last slice_layers layers × first slice_kv_heads KV heads (global,
    shards offset); the shared selection on Â reduces to the per-row selection when every
    row carries the same A (Â is then |slice|·A, the same order)."""
    assert msve.slice_rows(2, 4, 0, 0, 2, 0, 0) is None
    assert msve.slice_rows(2, 4, 0, 0, 4, 1, 2) == set()                     # layers 0-1 of 4
    assert msve.slice_rows(2, 4, 2, 4, 4, 1, 6) == {(1, 0), (1, 1)}          # shard: layers 2-3, heads 4-7
    tree, o, E = _small_state(levels=3, width=2, t_node=14, L=2, H=2, seed=21,
                              params=default_params(k_min=2, l_tail=3, r_min=0.0, select_shared=1))
    tree2, o2, _ = _small_state(levels=3, width=2, t_node=14, L=2, H=2, seed=21)
    rng = np.random.default_rng(5)
    base = rng.random(o.Tmax).astype(np.float32)
    A = np.broadcast_to(base, (2, 2, o.Tmax)).copy()
    tree.active = tree2.active = [synth.leaves_of(tree)[0]]
    k = [max(2, x // 3) for x in o.n]
    o.evict(tree, k, A_f32=A)
    o2.evict(tree2, k, A_f32=A)
    for i in range(len(o.n)):
        assert np.array_equal(o.kept[i], o2.kept[i])


# ---------------------------------------------------------------- f3 θ-fitter
def test_theta_fitter_gradient_constant_fit_and_separable():
    """The fitter's gradient equals a central finite difference of its loss (independent
    of the analytic formula); constant targets c converge to σ(θ₀) ≈ c; separable data
    (critical blocks v = 1) rank perfectly; the loss never increases."""
    from oracle import calibrate as cal
    rng = np.random.default_rng(4)
    phi = [tuple(float(x) for x in rng.random(3)) for _ in range(40)]
    y = [float(x) for x in rng.random(40)]
    th = [0.3, -0.7, 1.1, 0.2]
    g = cal.grad(th, phi, y)
    for k in range(4):
        e = [0.0] * 4
        e[k] = 1e-6
        fd = (cal.loss([a + b for a, b in zip(th, e)], phi, y) -
              cal.loss([a - b for a, b in zip(th, e)], phi, y)) / 2e-6
        assert abs(fd - g[k]) < 1e-8
    th_c, (l0, l1) = cal.fit_theta(phi, [0.2] * 40, [0, 0, 0, 0], 3000, 4.0)
    assert l1 <= l0 and l1 < 1e-6
    assert abs(cal.sigmoid(th_c[0] + sum(th_c[k + 1] * np.mean([p[k] for p in phi]) for k in range(3))) - 0.2) < 1e-3
    crit = [i % 3 == 0 for i in range(30)]
    phi2 = [(1.0 if c else 0.0, float(rng.random()), float(rng.random())) for c in crit]
    th_s, _ = cal.fit_theta(phi2, [1.0 if c else 0.0 for c in crit], [0, 0, 0, 0], 500, 4.0)
    sc = [cal.sigmoid(th_s[0] + th_s[1] * v + th_s[2] * u + th_s[3] * a) for v, u, a in phi2]
    assert min(s for s, c in zip(sc, crit) if c) > max(s for s, c in zip(sc, crit) if not c)
    # loss trace never increases (one epoch at a time from the same start)
    th, prev = [0, 0, 0, 0], cal.loss([0, 0, 0, 0], phi, y)
    for _ in range(20):
        th, (_, cur) = cal.fit_theta(phi, y, th, 1, 8.0)
        assert cur <= prev
        prev = cur


def test_stream_analogue_closed_forms():
    """The sequence-flattened StreamingLLM analogue: on the active path
    root → ℓ the most recent W = 𝓑 − |open| − |sinks| tokens are kept whole blocks first from
    the leaf up, one block partially, plus the root's sinks; off-path blocks get 0."""
    parent = [-1, 0, 0, 1, 1, 3]
    n = [10, 20, 30, 40, 50, 60]
    opn = [False] * 6
    st, k, _ = tae.stream_targets(parent, 5, opn, n, 4, 4 + 60 + 40 + 7)
    assert st == 0 and k == [4, 7, 0, 40, 0, 60]              # leaf, node 3 whole, node 1 partial
    st, k, _ = tae.stream_targets(parent, 5, opn, n, 4, 10 ** 6)
    assert k == [10, 20, 0, 40, 0, 60]                          # the whole path, nothing else
    st, k, _ = tae.stream_targets(parent, 5, opn, n, 4, 4 + 60 + 40 + 20 + 3)
    assert k == [7, 20, 0, 40, 0, 60]                           # sinks + the root's last 3
    opn[5] = True
    st, k, mf = tae.stream_targets(parent, 5, opn, n, 4, 50)
    assert st == 3 and mf == 64                                 # open leaf + sinks > 𝓑
    st, k, _ = tae.stream_targets(parent, 5, opn, n, 4, 64 + 5)
    assert k == [4, 0, 0, 5, 0, 60]
