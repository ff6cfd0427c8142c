"""f1 — the event-driven controller oracle (oracle/controller.py, Alg. 2) pinned by
what the paper fixes about the event loop, on synthetic Tree-of-Thoughts traces run fully on
the CPU oracle:
  * active-path protection after every handler: ∀ i ∈ Path*: k_i = n_i  (§3 (i), P:104;
    Alg. 2 l.8-14)
  * budget safety: Σ k ≤ 𝓑 after every Pressure  (Alg. 2 l.26-30; §3 PUE (iii) P:115)
  * Boundary touches only the closing block  ("of that block only")
  * Transition never grows an off-path retained set; rehydration happens only at Transition
    for blocks entering Path*  (Alg. 2 l.16-21, l.8-14; "only at that time")
  * FullKV (unlimited budget and α → ∞, so Eq. 2 gives r = 1 for every block) → no eviction,
    no Pressure, no rehydration
  * waterline: a Pressure is raised exactly when Σ k ≥ 𝓑 − δ, and never while one is
    pending  (Alg. 2 l.31-33)
  * determinism: the same seeded trace gives the same event log twice."""
from __future__ import annotations

import numpy as np
import pytest

import synth
from oracle import geometry, tae
from oracle.controller import ControllerOracle
from oracle.state import ArborOracle, default_params

SHAPE = dict(L=1, H=1, Hq=2, d=16, P=4)


def run_trace(seed=0, budget=None, delta=8, expansions=7, t_node=10, width=2, max_depth=3,
              mode=tae.MODE_WATERFILL, check=None, alpha=1.0):
    """A ToT search on the oracle: root prompt, then `expansions` times: pick a block to
    expand (∝ v), open a child there (Transition), decode t_node tokens into it (attention +
    score each step, waterline after each), close it (Boundary).  `check(event, ctl, tree,
    before)` runs after every handler with the per-node k_cur before it."""
    rng = np.random.default_rng(seed)
    tree = synth.full_tree(1, width, t_node, seed)          # the root (prompt) only
    T = t_node * (expansions + 1) + 4
    K, V, E = synth.make_kv(SHAPE["L"], SHAPE["H"], T, SHAPE["d"], "f32", seed,
                            tree.span_start, tree.span_len)
    params = default_params(k_min=2, l_tail=2, alloc_mode=mode, alpha=alpha)
    orc = ArborOracle(K.double().numpy(), V.double().numpy(), SHAPE["Hq"], SHAPE["P"],
                      4 * T // SHAPE["P"] + 8, params)
    orc.open_node(0, 0)
    orc.append(0, int(tree.span_len[0]))
    orc.close_node(0)
    big = budget is None
    ctl = ControllerOracle(orc, 10 ** 9 if big else budget, delta)
    tree.active = [0]
    step = [0]

    def decode():
        q = synth.make_queries(1, SHAPE["L"], SHAPE["Hq"], SHAPE["d"], "f32", 1000 + step[0], E)
        step[0] += 1
        orc.score_accumulate(tree, q.double().numpy())
        return orc.msve(tree)[1]

    def handle(kind, fn, *args):
        before = [orc.k_cur(i) for i in range(len(orc.n))]
        fn(*args)
        if check:
            check(kind, ctl, tree, before)

    s = decode()
    handle("boundary", ctl.boundary, tree, 0, s)
    next_pos = int(tree.span_len[0])
    for _ in range(expansions):
        pick = synth.tot_expansion(tree, rng, width, max_depth)
        if pick is None:
            break
        parent, v, u = pick
        child = tree.add_node(parent, next_pos, 0, True, v, u)
        orc.open_node(child, next_pos)
        next_pos += t_node
        tree.active = [child]
        handle("transition", ctl.transition, tree, orc.s_last)
        if ctl.waterline():
            handle("pressure", ctl.pressure, tree, orc.s_last)
        for _t in range(t_node):
            orc.append(child, 1)
            tree.span_len[child] += 1
            s = decode()
            if ctl.waterline():
                handle("pressure", ctl.pressure, tree, s)
        orc.close_node(child)
        tree.is_open[child] = 0
        s = orc.msve(tree)[1]
        handle("boundary", ctl.boundary, tree, child, s)
        if ctl.waterline():
            handle("pressure", ctl.pressure, tree, s)
    return ctl, orc, tree


def _path_full(ctl, tree):
    orc = ctl.orc
    for x in geometry.root_path(tree.parent, tree.active[0]):
        if not orc.open[x]:
            assert orc.k_cur(x) == orc.n[x], f"Path* node {x} not full"


@pytest.mark.parametrize("mode", [tae.MODE_WATERFILL, tae.MODE_STATIC_DRAIN])
def test_invariants_on_tot_traces(mode):
    seen = {"pressure": 0, "rehydrate": 0}

    def check(kind, ctl, tree, before):
        orc = ctl.orc
        _path_full(ctl, tree)
        after = [orc.k_cur(i) for i in range(len(orc.n))]
        _, _, on = orc.geometry(tree)
        if kind == "boundary":
            i = ctl.log[-1][1]
            assert all(after[j] == before[j] for j in range(len(before)) if j != i)
        if kind == "transition":
            grown = [j for j in range(len(before)) if after[j] > before[j]]
            assert all(on[j] for j in grown), "Transition grew an off-path block"
            seen["rehydrate"] += len(grown)
        if kind == "pressure":
            seen["pressure"] += 1
            assert ctl.total() <= ctl.budget, "Pressure left Σ k above the budget"
            assert all(after[j] <= before[j] for j in range(len(before)))
        if kind != "transition":
            assert all(after[j] <= before[j] for j in range(len(before))), f"{kind} grew a block"

    for seed in range(3):
        run_trace(seed=seed, budget=50, delta=6, mode=mode, check=check)
    assert seen["pressure"] > 0 and seen["rehydrate"] > 0


def test_full_kv_never_evicts_pressures_or_rehydrates():
    def check(kind, ctl, tree, before):
        assert kind != "pressure"
        orc = ctl.orc
        assert all(orc.k_cur(i) == orc.n[i] for i in range(len(orc.n))), "FullKV evicted"

    ctl, orc, _ = run_trace(seed=5, budget=None, check=check, alpha=1e9)
    assert orc.rehydrations == 0
    assert not any(e[0] == "pressure" for e in ctl.log)


def test_boundary_is_eq2_eq3_for_that_block():
    """With no budget pressure, after Boundary(i) the closing block keeps exactly the
    Eqs. 2-3 count computed from the same scores and geometry."""
    got = []

    def check(kind, ctl, tree, before):
        if kind != "boundary":
            return
        orc = ctl.orc
        i = ctl.log[-1][1]
        d, dist, on = orc.geometry(tree)
        _, k, _ = tae.allocate(tae.MODE_STATIC, orc.s_last, d, dist, on, orc.open, orc.n,
                               orc.params, 10 ** 9)
        assert orc.k_cur(i) == min(before[i], k[i])
        got.append((i, k[i], orc.n[i]))

    run_trace(seed=2, budget=None, check=check)
    assert any(k < n for _, k, n in got) or all(k == n for _, k, n in got)
    assert len(got) >= 2


def test_waterline_single_pending_and_threshold():
    orc_ctl, orc, _ = run_trace(seed=1, budget=10 ** 9, expansions=2)
    ctl = ControllerOracle(orc, budget=orc_ctl.total() + 5, delta=5)   # Σ k = 𝓑 − δ exactly
    assert ctl.waterline() is True
    assert ctl.waterline() is False          # pending: no second event
    ctl.pending = False
    ctl.budget += 1                          # Σ k = 𝓑 − δ − 1
    assert ctl.waterline() is False


def test_same_trace_same_log():
    a = run_trace(seed=4, budget=50, delta=6)[0].log
    b = run_trace(seed=4, budget=50, delta=6)[0].log
    assert a == b
