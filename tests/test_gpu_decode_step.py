"""GPU parity of f2, arbor_decode_step (include/arbor.h): decode attention + score as two
launches (attention kernel, then merge + score + masses + MSVE in one kernel; SURVEY §8(f)
f2).  Checked against the CPU oracle like the two-call path (tests in
test_gpu_parity.py), against the two-call path itself, and at the full sizes of configs[1],
configs[3] and configs[4] (8B-shaped 19,968 tokens; 32B-shaped 64 layers, G = 5, depth 8;
64k tokens) on sampled (layer, KV-head) rows, each mirrored by an oracle over that row alone.
"""
import math

import numpy as np
import pytest
import torch

import synth
from oracle.state import ArborOracle
from paper_2605_22106_b200 import workload

from gpu_helpers import Pair, assert_close, oracle_params
from test_gpu_parity import MID, _evict_both, _score_stage_checks

pytestmark = pytest.mark.gpu


def test_c1_decode_step_pipeline():
    """configs[0] (fp32, d = 64: the CUDA-core attention kernel feeds the fused merge+score)."""
    pr = Pair(workload.PRESETS["c1"], 0)
    pr.warmup(check=True, fused=True)
    pr.tree.active = [3]
    pr.decode_both(check=True, fused=True)
    sc = _score_stage_checks(pr)
    B = int(math.floor(0.5 * pr.tree.total_tokens))
    st, k_ref, _ = pr.discrete_allocate(sc["s"], B)
    assert st == 0 and sum(k_ref) == B
    _evict_both(pr, k_ref)
    pr.tree.active = [6]
    pr.ctx.arbor_rehydrate(pr.tree, [0, 2, 6])
    pr.orc.rehydrate([0, 2, 6])
    pr.check_kv_state()
    pr.decode_both(check=True, fused=True)
    _score_stage_checks(pr)


def test_mid_bf16_decode_step_after_evictions():
    """bf16 GQA on the tensor-core path; ragged 96-token nodes; decode over compacted pages."""
    pr = Pair(MID, seed=3)
    pr.warmup(steps_per_leaf=2, check=False, fused=True)
    pr.decode_both(check=True, fused=True)
    sc = _score_stage_checks(pr)
    B = int(0.25 * pr.tree.total_tokens)
    st, k_ref, _ = pr.discrete_allocate(sc["s"], B)
    _evict_both(pr, k_ref)
    pr.decode_both(check=True, fused=True)
    _score_stage_checks(pr)


def test_multi_leaf_decode_step_with_transitions():
    """4 active leaves sharing nodes (tiles with several leaves), then transitions with
    rehydration; every step through arbor_decode_step."""
    preset = dict(MID, tree=("full", 4, 3, 64), active="highest_v")
    pr = Pair(preset, seed=5, max_active=8)
    leaves = synth.leaves_of(pr.tree)
    pr.tree.active = leaves[:4]
    pr.decode_both(check=True, fused=True)
    sc = _score_stage_checks(pr)
    B = int(0.5 * pr.tree.total_tokens)
    st, k_ref, _ = pr.discrete_allocate(sc["s"], B)
    _evict_both(pr, k_ref)
    import oracle.geometry as g
    for t in range(2):
        pr.tree.active = leaves[4 * (t + 1): 4 * (t + 2)]
        path = sorted(set(x for l in pr.tree.active for x in g.root_path(pr.tree.parent, l)))
        pr.ctx.arbor_rehydrate(pr.tree, path)
        pr.orc.rehydrate(path)
        pr.decode_both(check=True, fused=True)
        _score_stage_checks(pr)


def test_decode_step_agrees_with_two_calls():
    """Same seeded scenario twice: arbor_decode_step vs arbor_tree_decode_attn + arbor_score.
    The merged LSE is summed in a different order (warp tree vs sequential), so floats agree
    to fp32 rounding, not bit for bit."""
    preset = dict(MID, tree=("full", 3, 4, 80))
    a = Pair(preset, seed=7, max_active=8)
    b = Pair(preset, seed=7, max_active=8)
    leaves = synth.leaves_of(a.tree)
    for step in range(6):
        act = [leaves[(3 * step + j) % len(leaves)] for j in range(1 + step % 3)]
        a.tree.active = act
        b.tree.active = act
        oa, la = a.decode_both(check=False, fused=True)
        ob, lb = b.decode_both(check=False, fused=False)
        assert_close(oa.float().cpu().numpy(), ob.float().cpu().numpy(), 8e-3, "out")
        assert_close(la.cpu().numpy(), lb.cpu().numpy(), 1e-6, "LSE")
    assert_close(a.gpu_A(), b.gpu_A(), 1e-5, "A", row_frac=1e-3)
    sa = a.ctx.arbor_read_scores(a.tree.num_nodes)
    sb = b.ctx.arbor_read_scores(b.tree.num_nodes)
    assert np.array_equal(sa["nq"], sb["nq"])
    assert np.allclose(sa["s"], sb["s"], rtol=1e-5, atol=1e-6)


@pytest.mark.parametrize("cfg", ["c2", "c4", "c5"])
def test_full_size_decode_step_sampled_rows(cfg):
    """configs[1] (c2), configs[3] (c4: Qwen2.5-32B-shaped, 64 layers, G = 5, depth-8 tree)
    and configs[4] (c5: 64k-token 8B-shaped tree) at full size in the bench's launch
    configuration: leaf-cycling warm-up, decode steps and a ρ = 0.25 eviction through
    arbor_decode_step / arbor_allocate / arbor_evict; sampled (layer, KV head) rows are
    mirrored by per-row oracles: attention output (2e-2), LSE and A (1e-5), kept positions,
    page lists and free list (bit-exact)."""
    preset = workload.PRESETS[cfg]
    sc = workload.setup(cfg, 0)
    ctx, tree = sc.ctx, sc.tree
    G = ctx.G
    Lm = ctx.L - 1
    rows = [(0, 0), (13, 5), (Lm, 7)]
    orcs = {}
    for (l, h) in rows:
        K = sc.K[l:l + 1, h:h + 1].double().cpu().numpy()
        V = sc.V[l:l + 1, h:h + 1].double().cpu().numpy()
        o = ArborOracle(K, V, G, ctx.P, ctx.NP, oracle_params(preset["params"]))
        for i in range(tree.num_nodes):
            o.open_node(i, int(tree.span_start[i]))
            o.append(i, int(tree.span_len[i]))
            o.close_node(i)
        orcs[(l, h)] = o
    nA = 1
    out = torch.empty((nA, ctx.L, ctx.Hq, ctx.D), dtype=torch.bfloat16, device="cuda")
    lse = torch.empty((nA, ctx.L, ctx.Hq), dtype=torch.float32, device="cuda")

    def step(check):
        q = sc.queries(sc.steps, nA)
        sc.steps += 1
        ctx.arbor_decode_step(tree, q, out, lse)
        for (l, h), o in orcs.items():
            qr = q[:, l:l + 1, h * G:(h + 1) * G].double().cpu().numpy()
            o_ref, l_ref = o.decode(tree, qr)
            o.score_accumulate(tree, qr, l_ref)
            if check:
                assert_close(out[:, l:l + 1, h * G:(h + 1) * G].float().cpu().numpy(), o_ref, 2e-2,
                             f"out row {(l, h)}")
                assert_close(lse[:, l:l + 1, h * G:(h + 1) * G].cpu().numpy(), l_ref, 1e-5,
                             f"LSE row {(l, h)}", row_frac=0.0)

    order = workload.leaf_cycle_order(tree, 0)
    for leaf in order[:40]:
        tree.active = [leaf]
        step(check=False)
    tree.active = [synth.highest_v_leaf(tree)]
    step(check=True)
    A = ctx.score
    for (l, h), o in orcs.items():
        assert_close(A[l, h, :o.Tmax].cpu().numpy()[None], o.A[0, 0][None], 1e-5, f"A row {(l, h)}",
                     row_frac=1e-3)
    s = torch.empty(tree.num_nodes, dtype=torch.float32, device="cuda")
    ctx.arbor_decode_step(tree, sc.queries(sc.steps, nA), out, lse, s)
    sc.steps += 1
    B = int(math.floor(preset["rho"] * tree.total_tokens))
    k = torch.empty(tree.num_nodes, dtype=torch.int32, device="cuda")
    ctx.arbor_allocate(tree, s, B, k)
    kl = k.cpu().tolist()
    assert sum(kl) == B
    ctx.arbor_evict(tree, k)
    Ah = A.cpu().numpy()
    free = ctx.arbor_read_free_list()
    for (l, h), o in orcs.items():
        o.evict(tree, kl, A_f32=Ah[l:l + 1, h:h + 1])
        assert o.free == free, "free list"
    for i in range(tree.num_nodes):
        kc, n, pages = ctx.arbor_read_node(i)
        ko = ctx.arbor_read_node_offset(i)
        idx = torch.as_tensor(pages, device="cuda", dtype=torch.long)
        for (l, h), o in orcs.items():
            assert kc == o.k_cur(i) and pages == o.pages[i] and ko == o.koff[i], i
            if kc:
                pos = ctx.pos_pool[l, idx, h].reshape(-1)[ko:ko + kc].cpu().numpy().astype(np.int64)
                assert np.array_equal(pos, o.kept[i][0, 0]), (i, (l, h))
    # decode over the compacted pages
    for leaf in order[40:44]:
        tree.active = [leaf]
        step(check=True)


def test_decode_step_without_lse_and_wide_fallback():
    """arbor_decode_step with lse_out = NULL (the merged LSE stays on chip only), and with
    more (leaf, q-head) pairs than the fused merge keeps on chip (65 leaves × G = 8 > 512:
    the call falls back to the two-call path) — both against the oracle."""
    preset = dict(tree=("full", 3, 9, 16), L=1, H=2, Hq=16, d=128, dtype="bf16", P=16, rho=0.5,
                  params={}, active="highest_v")
    pr = Pair(preset, seed=11, max_active=80)
    leaves = synth.leaves_of(pr.tree)
    # (1) lse_out = NULL
    pr.tree.active = leaves[:3]
    q = pr.queries(3)
    out = torch.empty_like(q.cuda())
    pr.ctx.arbor_decode_step(pr.tree, q.cuda(), out, None)
    o_ref, l_ref = pr.orc.decode(pr.tree, q.double().numpy())
    pr.orc.score_accumulate(pr.tree, q.double().numpy(), l_ref)
    assert_close(out.float().cpu().numpy(), o_ref, pr.rtol, "out (lse NULL)")
    _score_stage_checks(pr)
    # (2) 65 active leaves × 8 q heads: fallback
    pr.tree.active = leaves[:65]
    pr.decode_both(check=True, fused=True)
    _score_stage_checks(pr)
