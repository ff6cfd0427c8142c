"""configs[2] (C3, DPTS frontier) at FULL size: 16 active
leaves under distinct level-2 parents of the 8B-shaped depth-4 × width-5 tree (128-token
nodes, 32 layers, 8 KV heads, G = 4, bf16), ρ = 0.5 (𝓑 = 9,984 fixed while the tree grows),
transitions that replace 4 leaves (backtracks → rehydration), open children growing by decode
appends — in the bench's launch configuration (arbor_allocate / arbor_evict /
arbor_rehydrate / arbor_decode_step).  Sampled (layer, KV-head) rows are mirrored by per-row
oracles: k (tier (i), on the GPU's own s), kept positions, page lists, free list, K/V bytes
bit-exact; attention output (2e-2) and LSE / A (1e-5).  Plus: a 500-step stress of the
16-leaf decode (multi-leaf tensor-core tiles, two K stages) and of the 1-leaf C2 decode (three
K stages), and the ρ = 0.25 infeasibility with min_feasible = 120u + 1,248."""
import math

import numpy as np
import pytest
import torch

import synth
from oracle import tae
from oracle.state import ArborOracle
from paper_2605_22106_b200 import workload
from paper_2605_22106_b200.arbor import ArborError

from gpu_helpers import assert_close, oracle_params

pytestmark = pytest.mark.gpu

ROWS = [(0, 0), (13, 5), (31, 7)]


def test_c3_full_size_transitions_sampled_rows():
    T, D = 8, 8
    extra_nodes, extra_tokens, node_extra = workload.dpts_sizing(T, D)
    sc = workload.setup("c3", 0, extra_tokens=extra_tokens, extra_nodes=extra_nodes,
                        max_active=16, node_extra_tokens=node_extra)
    ctx, tree = sc.ctx, sc.tree
    preset = sc.preset
    G = ctx.G
    Ttot = tree.end_position() + extra_tokens
    orcs = {}
    for (l, h) in ROWS:
        K = np.zeros((1, 1, Ttot, ctx.D))
        V = np.zeros((1, 1, Ttot, ctx.D))
        K[:, :, :tree.end_position()] = sc.K[l:l + 1, h:h + 1].double().cpu().numpy()
        V[:, :, :tree.end_position()] = sc.V[l:l + 1, h:h + 1].double().cpu().numpy()
        o = ArborOracle(K, V, G, ctx.P, ctx.NP, oracle_params(preset["params"]))
        for i in range(tree.num_nodes):
            o.open_node(i, int(tree.span_start[i]))
            o.append(i, int(tree.span_len[i]))
            o.close_node(i)
        orcs[(l, h)] = o
    appended = {}

    def on_append(node, pos, k, v):
        appended[pos] = (k, v)
        for (l, h), o in orcs.items():
            o.K[0, 0, pos] = k[l, h, 0].double().numpy()
            o.V[0, 0, pos] = v[l, h, 0].double().numpy()

    # warm-up: 40 leaves of the seeded leaf cycle, one decode step each, mirrored
    out1 = torch.empty((1, ctx.L, ctx.Hq, ctx.D), dtype=torch.bfloat16, device="cuda")
    lse1 = torch.empty((1, ctx.L, ctx.Hq), dtype=torch.float32, device="cuda")
    for leaf in workload.leaf_cycle_order(tree, 0)[:40]:
        tree.active = [leaf]
        q = sc.queries(sc.steps, 1)
        sc.steps += 1
        ctx.arbor_decode_step(tree, q, out1, lse1)
        for (l, h), o in orcs.items():
            o.score_accumulate(tree, q[:, l:l + 1, h * G:(h + 1) * G].double().cpu().numpy())
    run = workload.DptsRun(sc, n_active=16, transitions=T, swap=4, decode_steps=D, seed=0,
                           on_append=on_append)
    o0 = orcs[ROWS[0]]
    rehyd_total = 0
    for t, leaves in enumerate([run.base_leaves] + run.schedule):
        n_log = len(run.log)
        kd = run.transition(leaves)
        for ev in run.log[n_log:]:
            for o in orcs.values():
                if ev[0] == "append":
                    o.append(ev[1], 1)
                elif ev[0] == "close":
                    o.close_node(ev[1])
                else:
                    o.open_node(ev[1], ev[2])
        s_gpu = ctx.arbor_read_scores(tree.num_nodes)["s"]
        d, dist, on_path = o0.geometry(tree)
        st, k_ref, _ = tae.allocate(o0.params["alloc_mode"], [float(x) for x in s_gpu], d, dist,
                                    on_path, o0.open, o0.n, o0.params, run.budget)
        assert st == 0 and kd.cpu().tolist() == k_ref, f"transition {t}: k differs"
        Ah = ctx.score.cpu().numpy()
        path = [x for x in run.path_union() if not tree.is_open[x]]
        for (l, h), o in orcs.items():
            rehyd = o.rehydrate(path)                   # Alg. 2: rehydrate, then evict
            o.evict(tree, k_ref, A_f32=Ah[l:l + 1, h:h + 1])
        rehyd_total += rehyd
        assert ctx.arbor_read_counters()[0] == o0.rehydrations
        free = ctx.arbor_read_free_list()
        for o in orcs.values():
            assert o.free == free, f"transition {t}: free list"
        for i in range(tree.num_nodes):
            kc, n, pages = ctx.arbor_read_node(i)
            ko = ctx.arbor_read_node_offset(i)
            if kc == 0:
                assert all(o.k_cur(i) == 0 for o in orcs.values())
                continue
            idx = torch.as_tensor(pages, device="cuda", dtype=torch.long)
            for (l, h), o in orcs.items():
                assert kc == o.k_cur(i) and pages == o.pages[i] and ko == o.koff[i], (t, i)
                pos = ctx.pos_pool[l, idx, h].reshape(-1)[ko:ko + kc].cpu().numpy().astype(np.int64)
                assert np.array_equal(pos, o.kept[i][0, 0]), (t, i, (l, h))
                if i % 7 == 0 or tree.is_open[i]:    # K/V bytes on a sample of nodes
                    kr = ctx.k_pool[l, idx, h].reshape(-1, ctx.D)[ko:ko + kc]
                    want = torch.as_tensor(o.K[0, 0, int(tree.span_start[i]) + pos]).to(torch.bfloat16)
                    assert torch.equal(kr.cpu().view(torch.int16), want.view(torch.int16)), (t, i)
        for _ in range(D):
            n_log = len(run.log)
            q, (out, lse) = run.decode()
            for ev in run.log[n_log:]:
                for o in orcs.values():
                    o.append(ev[1], 1)
            for (l, h), o in orcs.items():
                qr = q[:, l:l + 1, h * G:(h + 1) * G].double().cpu().numpy()
                o_ref, l_ref = o.decode(tree, qr)
                o.score_accumulate(tree, qr, l_ref)
                assert_close(out[:, l:l + 1, h * G:(h + 1) * G].float().cpu().numpy(), o_ref, 2e-2,
                             f"C3 full out row {(l, h)}")
                assert_close(lse[:, l:l + 1, h * G:(h + 1) * G].cpu().numpy(), l_ref, 1e-5,
                             f"C3 full LSE row {(l, h)}", row_frac=0.0)
        A = ctx.score
        for (l, h), o in orcs.items():
            assert_close(A[l, h, :o.Tmax].cpu().numpy()[None], o.A[0, 0][None], 1e-5,
                         f"C3 full A row {(l, h)}", row_frac=1e-3)
            for ch in tree.active:     # open children: no mass from their own queries
                a0 = int(tree.span_start[ch])
                assert not o.A[0, 0, a0:a0 + int(tree.span_len[ch])].any()
    assert rehyd_total > 0


def test_c3_rho_quarter_is_infeasible_with_min_feasible():
    """SURVEY §8(d) C3 / Appendix A 'Feasibility' (tests/golden c3_infeasible): at ρ = 0.25
    (𝓑 = 4,992) the pinned union of the 16 paths plus the off-path floors exceeds the budget:
    ARBOR_ERR_INFEASIBLE_BUDGET with min_feasible = 128u + 8(156 − u) = 120u + 1,248."""
    extra_nodes, extra_tokens, node_extra = workload.dpts_sizing(2, 8)
    sc = workload.setup("c3", 0, extra_tokens=extra_tokens, extra_nodes=extra_nodes,
                        max_active=16, node_extra_tokens=node_extra)
    run = workload.DptsRun(sc, n_active=16, transitions=2, swap=4, decode_steps=8, seed=0)
    B = int(math.floor(0.25 * 19968))
    assert B == 4992
    for leaves in [run.base_leaves] + run.schedule[:2]:
        run.activate(leaves)
        tree = sc.tree
        u = len([x for x in run.path_union() if x < 156])      # base-tree nodes on Path*
        assert u in (37, 38)
        k = run.k_buf[:tree.num_nodes]
        with pytest.raises(ArborError) as ei:
            sc.ctx.arbor_allocate(tree, None, B, k)
        assert ei.value.status == 3
        open_tokens = sum(int(tree.span_len[x]) for x in tree.active)
        # closed children of earlier transitions (n ≥ 1 token) add their floors min(n, 8)
        extra = sum(min(int(tree.span_len[x]), 8) for x in range(156, tree.num_nodes)
                    if not tree.is_open[x])
        assert ei.value.min_feasible == 120 * u + 1248 + open_tokens + extra
        for ch in tree.active:               # decode one token into every open child
            run._append(ch)


@pytest.mark.parametrize("cfg,steps", [("c3", 500), ("c2", 500)])
def test_decode_stress(cfg, steps):
    """Repeated arbor_decode_step on the full-size tree: the 16-leaf C3 frontier (tiles of up
    to 6 leaves, NQ = 32, two K stages) and the 1-leaf C2 step (NQ = 8, three K stages) —
    the pipelines whose mbarrier parity aliasing deadlocked in round 1 (attn_tc kcons).  The
    output must equal the first step's bit for bit (deterministic kernels; A grows, the
    attention does not depend on it)."""
    sc = workload.setup(cfg, 0)
    ctx, tree = sc.ctx, sc.tree
    nA = len(tree.active)
    q = sc.queries(0, nA)
    out = torch.empty_like(q)
    lse = torch.empty((nA, ctx.L, ctx.Hq), dtype=torch.float32, device="cuda")
    ref = None
    for i in range(steps):
        ctx.arbor_decode_step(tree, q, out, lse)
        if i == 0:
            torch.cuda.synchronize()
            ref = (out.clone(), lse.clone())
        if i % 100 == 99:
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    assert torch.equal(out.view(torch.int16), ref[0].view(torch.int16))
    assert torch.equal(lse, ref[1])
    ctx.arbor_sync()
