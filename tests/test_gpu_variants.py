"""f4 — policy variants as kernel modes against the oracle, bit-exact:
intra-block retention Tail-only and Sinks + Tail (arbor_params.select_mode) through two
successive evictions (the second acting on already-compacted blocks), and the no-rehydration
ablation (arbor_params.no_rehydrate: Transition/rehydrate leave evicted blocks partial).
MSVE-only (λ_d = λ_Δ = 0, η = 1) and TAE-only (constant s) are parameter settings of the
method's path: their allocations and the evictions after them are checked bit-exact at the end
(and pinned on the CPU in test_oracle_pins.test_ablation_variants_msve_only_and_tae_only)."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import synth

from gpu_helpers import Pair

pytestmark = pytest.mark.gpu

MID = dict(tree=("full", 3, 4, 56), L=2, H=2, Hq=8, d=128, dtype="bf16", P=16, rho=0.25,
           params={}, active="highest_v")


def _evict_both(pr, k):
    kd = torch.as_tensor(np.asarray(k, np.int32), device="cuda")
    ev = pr.ctx.arbor_evict(pr.tree, kd, want_count=True)
    assert ev == pr.orc.evict(pr.tree, k, A_f32=pr.gpu_A())
    pr.check_kv_state()


@pytest.mark.parametrize("mode", ["tail", "sinks_tail", "heavy"])
def test_select_mode_two_stage_eviction(mode):
    pr = Pair(MID, seed=5, params_over=dict(select_mode=mode, n_sinks=5, l_tail=6))
    pr.warmup(steps_per_leaf=1)
    N = pr.tree.num_nodes
    rng = np.random.default_rng(9)
    n = [int(x) for x in pr.tree.span_len]
    k1 = [int(rng.integers(n[i] // 3, n[i] + 1)) for i in range(N)]
    _evict_both(pr, k1)
    k2 = [int(rng.integers(0, k1[i] + 1)) for i in range(N)]
    _evict_both(pr, k2)
    if mode != "heavy":   # closed form on a node evicted from full retention
        j = next(i for i in range(N) if pr.orc.k_cur(i) > 8 and pr.orc.k_cur(i) < n[i])
        kc = pr.orc.k_cur(j)
        kept = sorted(int(x) for x in pr.orc.kept[j][0, 0])
        tl = min(6, n[j])
        # global sinks live in the root only; elsewhere Sinks + Tail = Tail-only
        sk = min(5, kc - tl) if (mode == "sinks_tail" and j == 0) else 0
        assert kept == sorted(set(range(sk)) | set(range(n[j] - (kc - sk), n[j])))
    pr.tree.active = [synth.leaves_of(pr.tree)[-1]]
    pr.decode_both()


def test_no_rehydrate_keeps_evicted_path_partial():
    pr = Pair(MID, seed=6, params_over=dict(no_rehydrate=True))
    pr.warmup(steps_per_leaf=1)
    N = pr.tree.num_nodes
    _evict_both(pr, [4] * N)
    leaf = synth.leaves_of(pr.tree)[0]
    pr.tree.active = [leaf]
    path = [x for x in range(N) if pr.orc.k_cur(x) < int(pr.tree.span_len[x])]
    pr.ctx.arbor_rehydrate(pr.tree, path)
    assert pr.orc.rehydrate(path) == 0
    pr.check_kv_state()
    assert pr.ctx.arbor_read_counters()[0] == 0
    pr.decode_both()       # attention over the partial Path* blocks


@pytest.mark.parametrize("mode", ["heavy", "sinks_tail"])
def test_k_protect_path_floor_and_global_sinks(mode):
    """Invariant (i) with the high floor (params.k_protect): Path* blocks — the root
    included — are allocated and evicted down to min(n, k_protect) instead of being pinned;
    the global sinks (the root's first n_sinks positions) survive every
    eviction of the root.  Bit-exact against the oracle (allocation on the GPU's s, selection
    on the GPU's A); then the controller's protected Transition rehydrates only blocks below
    their floor."""
    pr = Pair(MID, seed=8, params_over=dict(select_mode=mode, n_sinks=4, l_tail=6, k_protect=20))
    pr.warmup(steps_per_leaf=1)
    pr.decode_both()
    sc = pr.ctx.arbor_read_scores(pr.tree.num_nodes)
    N = pr.tree.num_nodes
    n = [int(x) for x in pr.tree.span_len]
    B = int(0.2 * sum(n))
    st, k_ref, _ = pr.discrete_allocate(sc["s"], B)
    assert st == 0 and sum(k_ref) == B
    k = torch.empty(N, dtype=torch.int32, device="cuda")
    pr.ctx.arbor_allocate(pr.tree, torch.as_tensor(sc["s"], device="cuda"), B, k)
    assert k.cpu().tolist() == k_ref
    d, dist, on = pr.orc.geometry(pr.tree)
    for j in range(N):
        if on[j]:
            assert k_ref[j] >= min(n[j], 20)
    assert k_ref[0] < n[0], "the root must be evicted for the sinks to matter"
    _evict_both(pr, k_ref)
    root = set(int(x) for x in pr.orc.kept[0][0, 0])
    assert set(range(4)) <= root, "global sinks evicted"
    pr.decode_both()
    # a protected Transition: rehydrate only Path* blocks below min(n, k_protect)
    pr.tree.active = [synth.leaves_of(pr.tree)[-1]]
    kd = torch.empty(N, dtype=torch.int32, device="cuda")
    from oracle.controller import ControllerOracle
    co = ControllerOracle(pr.orc, B, 0)
    pr.ctx.arbor_policy_event(pr.tree, "transition", -1, B, kd)
    s_now = pr.ctx.arbor_read_scores(N)["s"]       # the library's last scores (decode above)
    co.transition(pr.tree, [float(x) for x in s_now], A_f32=pr.gpu_A())
    pr.check_kv_state()
    assert pr.ctx.arbor_read_counters()[0] == pr.orc.rehydrations


@pytest.mark.parametrize("mode", ["heavy", "sinks_tail"])
def test_sinks_outnumber_heavy_slots(mode):
    """The root's global sinks compete among themselves when fewer heavy-hitter slots than
    sinks remain (m = k − |tail| < n_sinks): HEAVY keeps the sinks with the largest ⟨A, t⟩
    (oracle/select.rank_key: sink first, then A, then position), SINKS_TAIL the most recent
    sinks.  Two rounds (the second from a compacted root with first_slot > 0), bit-exact."""
    pr = Pair(MID, seed=19, params_over=dict(select_mode=mode, n_sinks=12, l_tail=6,
                                             k_protect=1))
    pr.warmup(steps_per_leaf=1)
    pr.decode_both()
    N = pr.tree.num_nodes
    n = [int(x) for x in pr.tree.span_len]
    for m_heavy in (9, 3):
        k = [max(1, int(0.5 * x)) for x in n]
        k[0] = 6 + m_heavy                            # 9 then 3 heavy slots for 12 sinks
        for j in range(N):
            k[j] = min(k[j], pr.orc.k_cur(j))
        _evict_both(pr, k)
        root = [int(x) for x in pr.orc.kept[0][0, 0]]
        assert len([p for p in root if p < 12]) == m_heavy
        pr.decode_both()


@pytest.mark.parametrize("shared", [0, 1])
def test_thin_slice_a_i_and_shared_selection(shared):
    """Thin slice 𝓛 × 𝓗 (params.slice_layers / slice_kv_heads): a_i counts
    the slice rows' mass only, normalised by |𝓛|·|𝓗_q|; with select_shared (the
    paper-literal shared selection, Q1) every block is ranked once by the
    slice-summed Â and every row keeps the same positions.  Masses bit-exact (oracle node
    mass on the GPU's A over the slice rows), s against the oracle's fp64 MSVE, k and kept
    sets bit-exact (tier (i))."""
    from oracle import msve as omsve
    preset = dict(MID, L=3, H=4, Hq=16)
    pr = Pair(preset, seed=12, params_over=dict(slice_layers=2, slice_kv_heads=2,
                                                 select_shared=shared))
    assert pr.orc.slice == {(l, h) for l in (1, 2) for h in (0, 1)}
    pr.warmup(steps_per_leaf=1)
    pr.decode_both()
    N = pr.tree.num_nodes
    sc = pr.ctx.arbor_read_scores(N)
    A = pr.gpu_A()[:, :, :pr.orc.Tmax].astype(np.float64)
    for i in range(N):
        m = omsve.node_mass(A, int(pr.tree.span_start[i]), int(pr.tree.span_len[i]), pr.orc.slice)
        assert int(sc["mass"][i]) == m, i
    a_ref, s_ref = pr.orc.msve(pr.tree)
    assert np.allclose(sc["a"], a_ref, rtol=1e-6, atol=1e-7)
    assert np.allclose(sc["s"], s_ref, rtol=1e-5)
    B = int(0.3 * pr.tree.total_tokens)
    st, k_ref, _ = pr.discrete_allocate(sc["s"], B)
    assert st == 0
    _evict_both(pr, k_ref)
    if shared:
        for i in range(N):
            rows = [sorted(int(x) for x in pr.orc.kept[i][l, h]) for l in range(3) for h in range(4)]
            assert all(r == rows[0] for r in rows), f"node {i}: rows keep different positions"
    pr.decode_both()


def test_stream_analogue_irreversible():
    """The flattened StreamingLLM analogue (alloc_mode STREAM) with irreversible
    eviction (no_rehydrate): allocation and eviction bit-exact against the oracle on
    one path, then after a backtrack to another leaf (the old path's blocks leave the stream
    for good); decode over what is left."""
    pr = Pair(MID, seed=14, params_over=dict(alloc_mode="stream", l_tail=0,
                                              select_mode="sinks_tail", n_sinks=4,
                                              no_rehydrate=True))
    pr.warmup(steps_per_leaf=1)
    leaves = synth.leaves_of(pr.tree)
    N = pr.tree.num_nodes
    for leaf, frac in ((leaves[0], 0.08), (leaves[-1], 0.06)):
        pr.tree.active = [leaf]
        pr.decode_both()
        B = int(frac * pr.tree.total_tokens)
        st, k_ref, _ = pr.discrete_allocate([0.5] * N, B)
        assert st == 0 and sum(k_ref) <= B
        k = torch.empty(N, dtype=torch.int32, device="cuda")
        pr.ctx.arbor_allocate(pr.tree, None, B, k)
        assert k.cpu().tolist() == k_ref
        _evict_both(pr, k_ref)
        path = [x for x in range(N) if pr.orc.k_cur(x) < int(pr.tree.span_len[x])]
        pr.ctx.arbor_rehydrate(pr.tree, path)      # a no-op under no_rehydrate
        assert pr.orc.rehydrate(path) == 0
        pr.check_kv_state()
    assert set(range(4)) <= set(int(x) for x in pr.orc.kept[0][0, 0])
    pr.decode_both()


@pytest.mark.parametrize("variant", ["msve_only", "tae_only"])
def test_ablation_allocations_bit_exact(variant):
    """P:408-414 ablations as parameter settings: MSVE-only (λ_d = λ_Δ = 0,
    η = 1: the weight is s^γ alone) and TAE-only (s ≡ const: the tree alone).  The device
    allocation equals the oracle's bit for bit, and the eviction that follows matches it."""
    over = dict(lambda_d=0.0, lambda_delta=0.0, eta=1.0) if variant == "msve_only" else \
        dict(lambda_d=0.0, lambda_delta=0.7, eta=1.0)
    pr = Pair(MID, seed=21, params_over=over)
    pr.warmup(steps_per_leaf=1, check=False, fused=True)
    N = pr.tree.num_nodes
    if variant == "msve_only":
        s = np.asarray(pr.ctx.arbor_read_scores(N)["s"], np.float32)
    else:
        s = np.full(N, 0.5, np.float32)
    B = int(0.3 * pr.tree.total_tokens)
    k = torch.empty(N, dtype=torch.int32, device="cuda")
    pr.ctx.arbor_allocate(pr.tree, torch.as_tensor(s, device="cuda"), B, k)
    st, k_ref, _ = pr.discrete_allocate(s, B)
    assert st == 0 and k.cpu().tolist() == k_ref and sum(k_ref) == B
    _evict_both(pr, k_ref)
