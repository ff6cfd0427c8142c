"""a4 (TAE allocation) at scale: 10,000+ random instances — random trees (2-60 nodes), random
active sets, open blocks, f32 scores with exact zeros and ties, random Π (K_min, L_tail, r_min,
λ_d, α, γ, k_protect) and budgets from infeasible to full — in all three modes, bit-exact
against the oracle's exact-rational allocation (SURVEY §8(c).3 asks for ~10^4 instances).
Infeasible budgets must return ARBOR_ERR_INFEASIBLE_BUDGET with the oracle's min_feasible."""
import numpy as np
import pytest
import torch

import synth
from oracle import geometry, tae
from paper_2605_22106_b200 import workload
from paper_2605_22106_b200.arbor import ArborError, make_params

from gpu_helpers import oracle_params

pytestmark = pytest.mark.gpu

MODES = ("waterfill", "static", "static_drain")


def _tree(rng, N):
    parent = [-1] + [int(rng.integers(0, i)) for i in range(1, N)]
    n = rng.integers(1, 24, size=N).astype(np.int32)
    t = synth.SynthTree(np.array(parent, np.int32), np.zeros(N, np.int64), n,
                        np.zeros(N, np.uint8), rng.random(N).astype(np.float32),
                        rng.random(N).astype(np.float32), [])
    t.span_start = np.concatenate([[0], np.cumsum(n[:-1])]).astype(np.int64)
    # a few childless nodes are open blocks (still being generated)
    kids = set(parent[1:])
    leaves = [i for i in range(1, N) if i not in kids]
    for i in leaves:
        if rng.random() < 0.1:
            t.is_open[i] = 1
    return t


def test_allocation_ten_thousand_random_instances():
    rng = np.random.default_rng(2026)
    preset = dict(tree=None, L=1, H=1, Hq=1, d=64, dtype="f32", P=4, rho=0.5, params={},
                  active=None)
    done = infeasible = 0
    trees = 0
    while done < 10_000:
        trees += 1
        N = int(rng.integers(2, 61))
        tree = _tree(rng, N)
        n = [int(x) for x in tree.span_len]
        leaves = synth.leaves_of(tree)
        d_ = geometry.depths([int(x) for x in tree.parent])
        for mode in MODES:
            pd = dict(alloc_mode=mode, n_sinks=0, k_min=int(rng.integers(0, 5)),
                      l_tail=int(rng.integers(0, 5)), r_min=float(rng.choice([0.0, 0.05, 0.2])),
                      lambda_d=float(rng.choice([0.0, 0.2, -0.1])),
                      alpha=float(rng.choice([0.5, 1.0, 3.0])), gamma=float(rng.choice([1.0, 2.0, 3.0])),
                      k_protect=int(rng.choice([0, 0, 4, 12, 30])))
            ctx = workload.make_context(preset, tree, params=make_params(**pd), page_margin=8)
            # the context must know the nodes: open, fill (K/V content is irrelevant to a4), close
            K = torch.zeros((1, 1, tree.end_position() + 8, 64), device="cuda")
            workload.load_tree(ctx, tree, K, K)
            op = oracle_params(pd)
            k = torch.full((N,), -1, dtype=torch.int32, device="cuda")
            for rep in range(6):
                act = sorted(set(int(x) for x in rng.choice(leaves, size=int(rng.integers(1, min(4, len(leaves)) + 1)))))
                tree.active = act
                s = rng.random(N).astype(np.float32)
                s[rng.random(N) < 0.15] = 0.0
                s[rng.random(N) < 0.15] = s[0]
                parent = [int(x) for x in tree.parent]
                dist = geometry.delta(parent, act)
                ps = geometry.path_star(parent, act)
                on = [i in ps for i in range(N)]
                opn = [bool(x) for x in tree.is_open]
                for B in (int(rng.integers(0, sum(n) + 5)), sum(n) // 2, sum(n) // 4):
                    st, k_ref, mf = tae.allocate({"waterfill": 0, "static": 1, "static_drain": 2}[mode],
                                                 [float(x) for x in s], d_, dist, on, opn, n, op, B)
                    sd = torch.as_tensor(s, device="cuda")
                    if st != 0:
                        with pytest.raises(ArborError) as e:
                            ctx.arbor_allocate(tree, sd, B, k)
                        assert e.value.status == 3 and e.value.min_feasible == mf, (mode, B, mf)
                        infeasible += 1
                    else:
                        ctx.arbor_allocate(tree, sd, B, k)
                        got = k.cpu().tolist()
                        assert got == k_ref, (trees, mode, pd, act, B, got, k_ref)
                    done += 1
            ctx.arbor_sync()
            del ctx
    print(f"a4 random parity: {done} instances on {trees} trees, {infeasible} infeasible")


def test_allocation_large_trees_bitonic_path():
    """Trees above 256 nodes take the allocate kernel's bitonic largest-remainder selection
    (allocate.cu): bit-exact against the oracle on 24 instances of 257-700 nodes."""
    rng = np.random.default_rng(77)
    preset = dict(tree=None, L=1, H=1, Hq=1, d=64, dtype="f32", P=4, rho=0.5, params={},
                  active=None)
    done = 0
    for trial in range(8):
        N = int(rng.integers(257, 701))
        tree = _tree(rng, N)
        n = [int(x) for x in tree.span_len]
        leaves = synth.leaves_of(tree)
        d_ = geometry.depths([int(x) for x in tree.parent])
        pd = dict(alloc_mode="waterfill", n_sinks=0, k_min=int(rng.integers(0, 5)),
                  l_tail=int(rng.integers(0, 5)), r_min=float(rng.choice([0.0, 0.05])))
        ctx = workload.make_context(preset, tree, params=make_params(**pd), page_margin=8)
        K = torch.zeros((1, 1, tree.end_position() + 8, 64), device="cuda")
        workload.load_tree(ctx, tree, K, K)
        op = oracle_params(pd)
        k = torch.full((N,), -1, dtype=torch.int32, device="cuda")
        for rep in range(3):
            act = sorted(set(int(x) for x in rng.choice(leaves, size=2)))
            tree.active = act
            s = rng.random(N).astype(np.float32)
            parent = [int(x) for x in tree.parent]
            dist = geometry.delta(parent, act)
            ps = geometry.path_star(parent, act)
            on = [i in ps for i in range(N)]
            B = int(sum(n) * float(rng.choice([0.3, 0.5, 0.7])))
            st, k_ref, mf = tae.allocate(0, [float(x) for x in s], d_, dist, on,
                                         [bool(x) for x in tree.is_open], n, op, B)
            if st != 0:
                continue
            ctx.arbor_allocate(tree, torch.as_tensor(s, device="cuda"), B, k)
            assert k.cpu().tolist() == k_ref, (trial, rep, N, B)
            done += 1
        ctx.arbor_sync()
    assert done >= 12
