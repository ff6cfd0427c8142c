"""CUDA Graph capture of the hot path (include/arbor.h arbor_capture_begin / arbor_capture_end /
arbor_graph_launch; SURVEY §8(d) timing protocol: eager and graph-captured steps).

One step = arbor_decode_step (a9 + a2 + a3) → arbor_allocate (a1 + a4) → arbor_evict (a5 + a6),
the step bench.py times.  Captured once per active leaf and replayed from the same restored
state, it must leave exactly what the eager calls leave: outputs, LSE, scores, k, the K/V /
pos pools, A, every page list and the free list — bit for bit.  The eager path itself is
checked against the oracle in test_gpu_parity.py / test_gpu_decode_step.py.
"""
import numpy as np
import pytest
import torch

import synth

from gpu_helpers import Pair
from test_gpu_parity import MID

pytestmark = pytest.mark.gpu


def _state(pr):
    ctx = pr.ctx
    nodes = [ctx.arbor_read_node(i) for i in range(pr.tree.num_nodes)]
    offs = [ctx.arbor_read_node_offset(i) for i in range(pr.tree.num_nodes)]
    return (ctx.k_pool.clone(), ctx.v_pool.clone(), ctx.pos_pool.clone(), ctx.score.clone(),
            nodes, offs, ctx.arbor_read_free_list())


def _same_state(a, b):
    for x, y in zip(a[:4], b[:4]):
        assert torch.equal(x.view(torch.uint8) if x.dtype != torch.int16 else x,
                           y.view(torch.uint8) if y.dtype != torch.int16 else y)
    assert a[4] == b[4] and a[5] == b[5] and a[6] == b[6]


def test_graph_replay_equals_eager_step():
    pr = Pair(MID, seed=11)
    pr.warmup(steps_per_leaf=1, check=False, fused=True)
    ctx, tree = pr.ctx, pr.tree
    leaves = sorted(synth.leaves_of(tree), key=lambda x: -float(tree.v[x]))[:2]
    N = tree.num_nodes
    B = int(0.3 * tree.total_tokens)
    qs = [pr.queries(1).cuda() for _ in leaves]
    out = torch.empty_like(qs[0])
    lse = torch.empty((1, ctx.L, ctx.Hq), dtype=torch.float32, device="cuda")
    s = torch.empty(N, dtype=torch.float32, device="cuda")
    k = torch.empty(N, dtype=torch.int32, device="cuda")
    snap = (ctx.k_pool.clone(), ctx.v_pool.clone(), ctx.pos_pool.clone(), ctx.score.clone())
    ctx.arbor_save_state(1)

    def restore():
        ctx.k_pool.copy_(snap[0])
        ctx.v_pool.copy_(snap[1])
        ctx.pos_pool.copy_(snap[2])
        ctx.score.copy_(snap[3])
        ctx.arbor_load_state(1)

    def step(i):
        tree.active = [leaves[i]]
        ctx.arbor_decode_step(tree, qs[i], out, lse, s)
        ctx.arbor_allocate(tree, s, B, k)
        ctx.arbor_evict(tree, k)

    eager = []
    for i in range(2):
        restore()
        step(i)
        torch.cuda.synchronize()
        eager.append((out.clone(), lse.clone(), s.clone(), k.clone(), _state(pr)))
    graphs = []
    try:
        for i in range(2):
            restore()
            ctx.arbor_capture_begin()
            step(i)
            graphs.append(ctx.arbor_capture_end())
        # replay in both orders, twice: a replay may follow any other work
        for i in (1, 0, 0, 1):
            out.zero_(); lse.zero_(); s.zero_(); k.zero_()
            restore()
            ctx.arbor_graph_launch(graphs[i])
            torch.cuda.synchronize()
            e = eager[i]
            assert torch.equal(out.view(torch.int16), e[0].view(torch.int16))
            assert torch.equal(lse, e[1]) and torch.equal(s, e[2]) and torch.equal(k, e[3])
            _same_state(_state(pr), e[4])
        # the eager API still works after capture (host mirrors and staging intact)
        restore()
        step(0)
        torch.cuda.synchronize()
        assert torch.equal(k, eager[0][3])
        _same_state(_state(pr), eager[0][4])
    finally:
        for g in graphs:
            ctx.arbor_graph_destroy(g)


def test_capture_misuse_is_reported():
    pr = Pair(MID, seed=12)
    from paper_2605_22106_b200.arbor import ArborError
    with pytest.raises(ArborError):
        pr.ctx.arbor_capture_end()          # not capturing
    pr.ctx.arbor_capture_begin()
    with pytest.raises(ArborError):
        pr.ctx.arbor_capture_begin()        # already capturing
    g = pr.ctx.arbor_capture_end()          # an empty graph is a valid graph
    pr.ctx.arbor_graph_launch(g)
    pr.ctx.arbor_graph_destroy(g)
    pr.ctx.arbor_sync()
    assert np.isfinite(pr.ctx.score.float().sum().item())
