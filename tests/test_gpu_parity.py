"""GPU parity: libarbor (through the C ABI) against the CPU oracle, element by element.

Integer work (k, kept positions, page tables, free list, K/V bytes) must be bit-exact;
floats (attention output, LSE, accumulated attention, scores) within the north_star
tolerance (1e-5 relative fp32, 2e-2 relative bf16; definition in gpu_helpers.assert_close).
Discrete stages are checked on the GPU's own f32 A and s (SURVEY §8(c) tier (i)); the
float stages against the oracle's fp64 recomputation.
"""
import math

import numpy as np
import pytest
import torch

import synth
from oracle import msve as omsve, tae as otae
from oracle.state import OracleError
from paper_2605_22106_b200 import workload
from paper_2605_22106_b200.arbor import ArborError

from gpu_helpers import Pair, assert_close

pytestmark = pytest.mark.gpu

MID = dict(tree=("full", 4, 4, 96), L=2, H=4, Hq=16, d=128, dtype="bf16", P=16, rho=0.25,
           params={}, active="highest_v")


def _score_stage_checks(pr: Pair):
    """Float tier for A; exact tier for masses/s recomputed from the GPU's own A."""
    A = pr.gpu_A()[:, :, :pr.orc.Tmax]
    Aref = pr.orc.A
    assert_close(A, Aref, pr.rtol_q, "accumulated attention A", row_frac=1e-3)
    sc = pr.ctx.arbor_read_scores(pr.tree.num_nodes)
    A64 = A.astype(np.float64)
    for i in range(pr.tree.num_nodes):
        if pr.orc.open[i]:
            continue
        m = omsve.node_mass(A64, int(pr.tree.span_start[i]), int(pr.tree.span_len[i]))
        assert int(sc["mass"][i]) == m, f"node {i} mass {sc['mass'][i]} != {m}"
        assert int(sc["nq"][i]) == pr.orc.Nq[i]
        a = omsve.attention_feature(m, int(sc["mclose"][i]), pr.orc.Nq[i], pr.ctx.L, pr.ctx.Hq)
        s = float(np.float32(omsve.msve_score(pr.orc.params["theta"], float(pr.tree.v[i]),
                                               float(pr.tree.u[i]), a)))
        assert abs(float(sc["a"][i]) - a) <= 1e-6 * max(1.0, a)
        assert abs(float(sc["s"][i]) - s) <= 2 ** -23, (i, sc["s"][i], s)
    # oracle's own fp64 masses: tolerance
    a_ref, s_ref = pr.orc.msve(pr.tree)
    assert_close(sc["s"][None], np.array(s_ref, np.float64)[None], 1e-5, "MSVE s vs fp64 oracle", row_frac=0.0)
    return sc


def _evict_both(pr: Pair, k):
    kd = torch.as_tensor(np.asarray(k, np.int32), device="cuda")
    ev = pr.ctx.arbor_evict(pr.tree, kd, want_count=True)
    ev_ref = pr.orc.evict(pr.tree, k, A_f32=pr.gpu_A())
    assert ev == ev_ref
    pr.check_kv_state()


@pytest.mark.parametrize("seed", [0, 1])
def test_c1_full_pipeline(seed):
    """configs[0] end to end: warm-up, decode, score, allocate (B = 112), evict, backtrack
    with rehydration, decode again — every stage against the oracle."""
    pr = Pair(workload.PRESETS["c1"], seed)
    pr.warmup(check=True)
    pr.tree.active = [3]
    pr.decode_both(check=True)
    sc = _score_stage_checks(pr)
    B = int(math.floor(0.5 * pr.tree.total_tokens))
    assert B == 112
    k = torch.empty(pr.tree.num_nodes, dtype=torch.int32, device="cuda")
    sd = torch.as_tensor(sc["s"], device="cuda")
    pr.ctx.arbor_allocate(pr.tree, sd, B, k)
    st, k_ref, _ = pr.discrete_allocate(sc["s"], B)
    assert st == 0 and k.cpu().tolist() == k_ref and sum(k_ref) == B
    _evict_both(pr, k_ref)
    # backtrack to the other subtree: Path* = {0, 2, 6}; nodes 2 and 6 were evicted
    pr.tree.active = [6]
    path = [0, 2, 6]
    pr.ctx.arbor_rehydrate(pr.tree, path)
    n_re = pr.orc.rehydrate(path)
    assert n_re >= 1
    pr.check_kv_state()
    assert pr.ctx.arbor_read_counters()[0] == pr.orc.rehydrations
    pr.decode_both(check=True)
    _score_stage_checks(pr)


def test_mid_bf16_pipeline_with_ties():
    """bf16 GQA (G = 4), 85 nodes, 96-token nodes (ragged vs 128-slot chunks and 16-slot
    pages); 2% of A overwritten with a neighbour's value to create exact key ties."""
    pr = Pair(MID, seed=3)
    pr.warmup(steps_per_leaf=2, check=False)
    pr.decode_both(check=True)
    sc = _score_stage_checks(pr)
    A = pr.ctx.score
    rng = np.random.default_rng(0)
    T = pr.tree.total_tokens
    idx = rng.choice(T - 1, size=max(1, T // 50), replace=False)
    A[:, :, idx] = A[:, :, idx + 1]
    pr.ctx.arbor_invalidate_masses()      # A written directly (include/arbor.h)
    B = int(0.25 * pr.tree.total_tokens)
    k = torch.empty(pr.tree.num_nodes, dtype=torch.int32, device="cuda")
    pr.ctx.arbor_allocate(pr.tree, torch.as_tensor(sc["s"], device="cuda"), B, k)
    st, k_ref, _ = pr.discrete_allocate(sc["s"], B)
    assert k.cpu().tolist() == k_ref and sum(k_ref) == B
    _evict_both(pr, k_ref)
    pr.decode_both(check=True)
    # a second, deeper eviction (incremental: k only shrinks, Q17) then full restore
    k2 = [max(0, x // 2) for x in k_ref]
    _evict_both(pr, k2)
    pr.decode_both(check=True)


def test_multi_leaf_sharing_and_transitions():
    """DPTS-style frontier (4 active leaves sharing the root and level-1 nodes): decode
    attention reads a shared node once for all leaves; after eviction, transitions
    rehydrate the new paths (lazy rehydration, Alg. 2)."""
    preset = dict(MID, tree=("full", 4, 3, 64), active="highest_v")
    pr = Pair(preset, seed=5, max_active=8)
    leaves = synth.leaves_of(pr.tree)
    pr.tree.active = leaves[:4]
    pr.decode_both(check=True)
    sc = _score_stage_checks(pr)
    B = int(0.5 * pr.tree.total_tokens)
    st, k_ref, _ = pr.discrete_allocate(sc["s"], B)
    _evict_both(pr, k_ref)
    for t in range(3):
        pr.tree.active = leaves[4 * (t + 1): 4 * (t + 2)] or leaves[-4:]
        import oracle.geometry as g
        path = sorted(set(x for l in pr.tree.active for x in g.root_path(pr.tree.parent, l)))
        pr.ctx.arbor_rehydrate(pr.tree, path)
        pr.orc.rehydrate(path)
        pr.check_kv_state()
        pr.decode_both(check=True)
        sc = _score_stage_checks(pr)
        st, k_ref, _ = pr.discrete_allocate(sc["s"], B)
        _evict_both(pr, k_ref)


def test_open_nodes_and_appends():
    """Open children (active leaves being decoded) grow by appends; they are pinned; close
    snapshots Mclose and stashes; the new node then takes part in eviction."""
    preset = dict(MID, tree=("full", 3, 3, 40))
    pr = Pair(preset, seed=7, extra_tokens=64, extra_nodes=2)
    leaf = synth.leaves_of(pr.tree)[2]
    a = pr.tree.end_position()
    node = pr.tree.add_node(leaf, a, 0, True, 0.7, 0.4)
    pr.ctx.arbor_open_node(node, a)
    pr.orc.open_node(node, a)
    pr.tree.active = [node]
    extraK, extraV, _ = synth.make_kv(pr.ctx.L, pr.ctx.H, 64, pr.ctx.D, pr.preset["dtype"], 99)
    pr.orc.K[:, :, a:a + 64] = extraK.double().numpy()
    pr.orc.V[:, :, a:a + 64] = extraV.double().numpy()
    pr.K[:, :, a:a + 64] = extraK
    pr.V[:, :, a:a + 64] = extraV
    for t in range(5):       # appends of 1, 2, 3, 4, 5 tokens
        nt = t + 1
        off = pr.tree.span_len[node]
        pr.ctx.arbor_append_kv(node, extraK[:, :, off:off + nt].contiguous().cuda(),
                               extraV[:, :, off:off + nt].contiguous().cuda())
        pr.orc.append(node, nt)
        pr.tree.span_len[node] += nt
        pr.decode_both(check=True)
        # A_i(t) = Σ_{u>b_i} (DESIGN Q5'): the open block gets nothing from its own queries
        assert not pr.gpu_A()[:, :, a:a + int(pr.tree.span_len[node])].any()
    pr.check_kv_state()
    sc = _score_stage_checks(pr)
    pr.ctx.arbor_close_node(node)
    pr.orc.close_node(node)
    pr.tree.is_open[node] = 0
    pr.decode_both(check=True)
    sc = _score_stage_checks(pr)
    B = int(0.5 * pr.tree.total_tokens)
    st, k_ref, _ = pr.discrete_allocate(sc["s"], B)
    assert st == 0
    _evict_both(pr, k_ref)


def test_allocation_random_trees_bit_exact():
    """a4 on random trees, all three modes, random f32 scores (incl. exact zeros and ties)
    — bit-exact k against the oracle's exact-rational allocation."""
    rng = np.random.default_rng(11)
    preset = dict(tree=None, L=1, H=1, Hq=1, d=64, dtype="f32", P=4, rho=0.5, params={},
                  active=None)
    for trial in range(12):
        N = int(rng.integers(2, 120))
        parent = [-1] + [int(rng.integers(0, i)) for i in range(1, N)]
        n = rng.integers(1, 24, size=N).astype(np.int32)
        tree = synth.SynthTree(np.array(parent, np.int32), np.zeros(N, np.int64), n,
                               np.zeros(N, np.uint8), rng.random(N).astype(np.float32),
                               rng.random(N).astype(np.float32), [])
        # spans: children after parents — pack in id order
        tree.span_start = np.concatenate([[0], np.cumsum(n[:-1])]).astype(np.int64)
        tree.active = [int(x) for x in rng.choice(N, size=int(rng.integers(1, min(4, N) + 1)), replace=False)]
        for mode in ("waterfill", "static", "static_drain"):
            pr = Pair(preset, seed=trial, tree=tree.copy(), params_over=dict(
                alloc_mode=mode, n_sinks=0, k_min=int(rng.integers(0, 4)), l_tail=int(rng.integers(0, 4)),
                r_min=float(rng.choice([0.0, 0.05])), lambda_d=float(rng.choice([0.0, 0.2, -0.1])),
                alpha=float(rng.choice([0.5, 1.0, 3.0]))))
            s = rng.random(N).astype(np.float32)
            s[rng.random(N) < 0.15] = 0.0
            s[rng.random(N) < 0.15] = s[0]
            mf = None
            for B in (int(rng.integers(0, n.sum() + 5)), int(n.sum() // 2), int(n.sum())):
                st, k_ref, mf = pr.discrete_allocate(s, B)
                k = torch.full((N,), -1, dtype=torch.int32, device="cuda")
                if st != 0:
                    with pytest.raises(ArborError) as e:
                        pr.ctx.arbor_allocate(pr.tree, torch.as_tensor(s, device="cuda"), B, k)
                    assert e.value.status == 3 and e.value.min_feasible == mf
                    continue
                pr.ctx.arbor_allocate(pr.tree, torch.as_tensor(s, device="cuda"), B, k)
                got = k.cpu().tolist()
                if got != k_ref:
                    import json
                    with open("gpurun_out/alloc_fail.json", "w") as f:
                        json.dump(dict(trial=trial, mode=mode, B=B, got=got, want=k_ref, s=[float(x) for x in s],
                                       n=n.tolist(), parent=parent, active=pr.tree.active,
                                       params=pr.params_dict), f)
                assert got == k_ref, (trial, mode, B, got, k_ref)
            pr.ctx.arbor_sync()


def test_edge_cases_and_errors():
    pr = Pair(workload.PRESETS["c1"], seed=2)
    pr.decode_both(check=True)
    sc = _score_stage_checks(pr)
    N = pr.tree.num_nodes
    k = torch.empty(N, dtype=torch.int32, device="cuda")
    # unlimited budget = full retention: evict is a no-op
    pr.ctx.arbor_allocate(pr.tree, torch.as_tensor(sc["s"], device="cuda"), 10 ** 9, k)
    assert k.cpu().tolist() == pr.tree.span_len.tolist()
    assert pr.ctx.arbor_evict(pr.tree, k, want_count=True) == 0
    # infeasible budget reports the minimum feasible one and changes nothing
    with pytest.raises(ArborError) as e:
        pr.ctx.arbor_allocate(pr.tree, None, 10, k)
    assert e.value.status == 3 and e.value.min_feasible == 96 + 4 * 2
    # k_target 0 and k <= L_tail branch (Alg. 1), pinned nodes untouched
    tgt = [0, 0, 0, 1, 2, 0, 1]
    _evict_both(pr, tgt)
    assert pr.ctx.arbor_read_node(0)[0] == 32      # root pinned
    # rehydrate: no-op on full nodes, error on an open node
    pr.ctx.arbor_rehydrate(pr.tree, [0, 1, 3])
    assert pr.orc.rehydrate([0, 1, 3]) == 0
    pr.check_kv_state()
    with pytest.raises(ArborError) as e:
        pr.ctx.arbor_close_node(0)
    assert e.value.status == 7
    # invalid trees
    bad = pr.tree.copy()
    bad.parent[2] = 5
    with pytest.raises(ArborError):
        pr.ctx.arbor_score(bad, torch.zeros(1, 1, 2, 64, device="cuda"))
    bad = pr.tree.copy()
    bad.span_len[4] = 31
    with pytest.raises(ArborError):
        pr.ctx.arbor_evict(bad, k)


def test_nan_score_is_an_invariant_error():
    """A NaN accumulated attention that would order heavy hitters is ARBOR_ERR_INVARIANT,
    latched by the kernel and surfaced at the next sync (include/arbor.h conventions)."""
    pr = Pair(workload.PRESETS["c1"], seed=2)
    N = pr.tree.num_nodes
    pr.ctx.score[0, 0, int(pr.tree.span_start[5])] = float("nan")   # non-tail slot of node 5
    pr.ctx.arbor_invalidate_masses()
    tgt = torch.tensor([32, 32, 32, 32, 32, 10, 32], dtype=torch.int32, device="cuda")
    pr.ctx.arbor_evict(pr.tree, tgt)     # node 5: k 32 -> 10 > L_tail: ranked by A
    with pytest.raises(ArborError) as e:
        pr.ctx.arbor_sync()
    assert e.value.status == 4
    pr.ctx.arbor_sync()                  # the latch is cleared once reported


def test_stash_rehydrate_bit_exact_roundtrip():
    """Evict everything evictable to 0, then rehydrate all: the pages hold the original K/V
    byte for byte with pos = identity (P:199 'the same conditioning state')."""
    pr = Pair(MID, seed=4)
    N = pr.tree.num_nodes
    zero = [0] * N
    _evict_both(pr, zero)
    allnodes = list(range(N))
    pr.ctx.arbor_rehydrate(pr.tree, allnodes)
    assert pr.orc.rehydrate(allnodes) > 0
    pr.check_kv_state()
    for i in range(N):
        kc, pages, pos, kr, vr, _ = pr.gpu_node(i)
        assert kc == int(pr.tree.span_len[i]) and np.array_equal(pos[0, 0], np.arange(kc))


def test_c3_dpts_transitions_reduced():
    """configs[2] shape at reduced size: 16 active leaves under distinct level-2 parents,
    transitions replacing 4 of them (backtracking → rehydration), open children growing by
    decode appends; every transition's k, kept sets, pages, free list and rehydration count
    bit-exact, decode outputs and scores within tolerance."""
    preset = dict(workload.PRESETS["c3"], tree=("full", 4, 5, 24), L=2, H=2, Hq=8, rho=0.7)
    T_extra, N_extra = (16 + 3 * 4) * (2 * 4 + 2) + 64, 16 + 4 * 4 + 4
    pr = Pair(preset, seed=3, extra_tokens=T_extra, extra_nodes=N_extra, max_active=16)
    sc = workload.Scenario(pr.preset, pr.tree, pr.ctx, pr.Kd, pr.Vd, pr.E, 3, 0)

    def on_append(node, pos, k, v):
        pr.orc.K[:, :, pos] = k[:, :, 0].double().numpy()
        pr.orc.V[:, :, pos] = v[:, :, 0].double().numpy()
        pr.K[:, :, pos] = k[:, :, 0]
        pr.V[:, :, pos] = v[:, :, 0]

    run = workload.DptsRun(sc, n_active=16, transitions=3, swap=4, decode_steps=2, seed=3,
                           on_append=on_append)
    pr.warmup(steps_per_leaf=1)
    for t, leaves in enumerate([run.base_leaves] + run.schedule):
        n_log = len(run.log)
        kd = run.transition(leaves)
        for ev in run.log[n_log:]:                      # replay lifecycle events in order
            if ev[0] == "append":
                pr.orc.append(ev[1], 1)
            elif ev[0] == "close":
                pr.orc.close_node(ev[1])
            else:
                pr.orc.open_node(ev[1], ev[2])
        sc_gpu = pr.ctx.arbor_read_scores(pr.tree.num_nodes)
        st, k_ref, _ = pr.discrete_allocate(sc_gpu["s"], run.budget)
        assert st == 0 and kd.cpu().tolist() == k_ref, f"transition {t}: k differs"
        path = [x for x in run.path_union() if not pr.tree.is_open[x]]
        pr.orc.rehydrate(path)                          # Alg. 2: rehydrate, then evict
        pr.orc.evict(pr.tree, k_ref, A_f32=pr.gpu_A())
        pr.check_kv_state()
        assert pr.ctx.arbor_read_counters()[0] == pr.orc.rehydrations
        for _ in range(run.decode_steps):
            n_log = len(run.log)
            q, (out, lse) = run.decode()
            for ev in run.log[n_log:]:
                pr.orc.append(ev[1], 1)
            qn = q.float().cpu().double().numpy()
            o_ref, lse_ref = pr.orc.decode(pr.tree, qn)
            pr.orc.score_accumulate(pr.tree, qn)
            assert_close(out.float().cpu().numpy(), o_ref, pr.rtol, "C3 attention output")
            assert_close(lse.cpu().numpy(), lse_ref, pr.rtol_q, "C3 LSE", row_frac=0.0)
        _score_stage_checks(pr)
    assert pr.orc.rehydrations > 0
