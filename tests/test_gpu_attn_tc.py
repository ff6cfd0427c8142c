"""GPU parity of the tcgen05 tensor-core tree decode attention (attn_tc.cu) against the CPU
oracle, element by element (north_star bf16 tolerance 2e-2 relative, gpu_helpers.assert_close).

Covers: ragged node lengths (a tile whose second 64-slot chunk is partial, or absent), page
tails past k_cur holding NaN bytes (the kernel must not let them into 0·v), 1 / 3 / 9 active
leaves sharing nodes (NQ = 16 / 32 / 48 variants), G = 4 and G = 5, eviction to ragged k, and
the fused score pass fed from the tensor-core logits.  The CUDA-core kernel (ARBOR_ATTN=cuda)
is run on the same scenario as a second, independent GPU path.
"""
import os

import numpy as np
import pytest
import torch

import synth
from paper_2605_22106_b200 import workload

from gpu_helpers import Pair, assert_close

pytestmark = pytest.mark.gpu

RAGGED = dict(tree=("full", 3, 3, 93), L=2, H=4, Hq=16, d=128, dtype="bf16", P=16, rho=0.4,
              params={}, active="highest_v")


def _poison_page_tails(pr: Pair):
    """Write NaN into every slot past the valid ones of each node's last page, and before
    them in its first page (an evicted node's valid slots start at first_slot, Q23*) —
    garbage by contract."""
    P = pr.ctx.P
    for i in range(pr.tree.num_nodes):
        kc, n, pages = pr.ctx.arbor_read_node(i)
        ko = pr.ctx.arbor_read_node_offset(i)
        if not pages:
            continue
        e = (ko + kc) % P
        if e:
            pr.ctx.k_pool[:, pages[-1], :, e:] = float("nan")
            pr.ctx.v_pool[:, pages[-1], :, e:] = float("nan")
        if ko:
            pr.ctx.k_pool[:, pages[0], :, :ko] = float("nan")
            pr.ctx.v_pool[:, pages[0], :, :ko] = float("nan")


def _evict_ragged(pr: Pair, frac: float):
    k = [max(0, int(frac * int(n)) - (i % 5)) for i, n in enumerate(pr.tree.span_len)]
    for x in set(x for l in pr.tree.active for x in _path(pr.tree.parent, l)):
        k[x] = int(pr.tree.span_len[x])           # Path* is pinned (Q19)
    kd = torch.as_tensor(np.asarray(k, np.int32), device="cuda")
    pr.ctx.arbor_evict(pr.tree, kd)
    pr.orc.evict(pr.tree, k, A_f32=pr.gpu_A())
    pr.check_kv_state()


def _path(parent, leaf):
    out = []
    while leaf >= 0:
        out.append(int(leaf))
        leaf = int(parent[leaf])
    return out


@pytest.mark.parametrize("Hq,n_active", [(16, 1), (16, 3), (16, 9), (20, 9)])
def test_tc_attention_ragged_shared_nan_tails(Hq, n_active):
    preset = dict(RAGGED, Hq=Hq)
    pr = Pair(preset, seed=11 + n_active, max_active=16)
    assert pr.ctx.arbor_attn_tensor_cores(), "tensor-core attention not enabled for bf16/d128"
    leaves = synth.leaves_of(pr.tree)
    pr.tree.active = leaves[:n_active]
    pr.decode_both(check=True)
    assert_close(pr.gpu_A()[:, :, :pr.orc.Tmax], pr.orc.A, pr.rtol_q, "A", row_frac=1e-3)
    # evict the off-path nodes to ragged k (partial chunks and partial pages), poison tails
    pr.tree.active = leaves[:1]
    _evict_ragged(pr, 0.55)
    _poison_page_tails(pr)
    pr.tree.active = leaves[:n_active]
    # rehydrate the active paths (Alg. 2 Transition) so that every node is visible again
    path = sorted(set(x for l in pr.tree.active for x in _path(pr.tree.parent, l)))
    pr.ctx.arbor_rehydrate(pr.tree, path)
    pr.orc.rehydrate(path)
    _poison_page_tails(pr)
    out, lse = pr.decode_both(check=True)
    assert torch.isfinite(out.float()).all()
    assert_close(pr.gpu_A()[:, :, :pr.orc.Tmax], pr.orc.A, pr.rtol_q, "A", row_frac=1e-3)


def test_tc_attention_evicted_nodes_visible():
    """Active leaves whose paths cross evicted (k_cur < n, ragged) nodes: chunks with 0 < nt <
    64, empty second chunks and NaN page tails are all read by the tensor-core kernel."""
    pr = Pair(RAGGED, seed=5, max_active=16)
    leaves = synth.leaves_of(pr.tree)
    pr.tree.active = leaves[:1]
    _evict_ragged(pr, 0.3)
    _poison_page_tails(pr)
    pr.tree.active = leaves[-4:]                   # paths over evicted nodes, no rehydration
    out, _ = pr.decode_both(check=True)
    assert torch.isfinite(out.float()).all()


def test_tc_matches_cuda_core_path():
    """Same scenario through both GPU kernels (independent code paths) and the oracle."""
    outs = []
    for mode in ("tc", "cuda"):
        if mode == "cuda":
            os.environ["ARBOR_ATTN"] = "cuda"
        try:
            pr = Pair(RAGGED, seed=21, max_active=16)
        finally:
            os.environ.pop("ARBOR_ATTN", None)
        assert pr.ctx.arbor_attn_tensor_cores() == (mode == "tc")
        pr.tree.active = synth.leaves_of(pr.tree)[:5]
        out, lse = pr.decode_both(check=True)
        outs.append((out.float().cpu().numpy(), lse.cpu().numpy(), pr.gpu_A()))
    assert_close(outs[0][0], outs[1][0], 2e-2, "tc vs cuda-core output")
    assert_close(outs[0][1], outs[1][1], 1e-5, "tc vs cuda-core LSE", row_frac=0.0)
    assert_close(outs[0][2], outs[1][2], 1e-5, "tc vs cuda-core A", row_frac=1e-3)
