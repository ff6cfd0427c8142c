"""Randomised select + compact (a5 + a6) and partial rehydration (a8) against the oracle.

Each trial draws a random tree (full, or DPTS-like best-first growth; node lengths off the
16-slot page and 64-slot chunk grid), writes a random accumulated-attention field A straight into the caller-owned score buffer — mixtures of
log-uniform magnitudes, exact zeros and heavily quantised values, so that many keys tie on A
and only the position breaks the tie (Q3), and the radix select meets every path: one digit
pass, several passes, the rank-count finish, whole-bin survival — and then runs, on both
sides, several rounds of: a random k (shrinking only, Q17, floors and k = 0 included) →
arbor_evict vs ArborOracle.evict on the same f32 A → bit-exact K/V bytes, pos tags, page lists
and free list; every other round a random set of evicted nodes is rehydrated (Q23r:
kept rows restored within HBM, the rest from the stash) and compared the same way.
"""
import numpy as np
import pytest
import torch

import synth
from paper_2605_22106_b200 import workload

from gpu_helpers import Pair

pytestmark = pytest.mark.gpu


def _random_A(rng, shape):
    A = np.exp(rng.uniform(-18.0, 2.0, size=shape)).astype(np.float32)
    kind = rng.integers(0, 4)
    if kind == 1:        # quantised: heavy ties within a row
        A = (np.round(A * 8.0) / 8.0).astype(np.float32)
    elif kind == 2:      # few distinct values per row
        A = rng.choice(np.float32([0.0, 0.5, 1.0, 3.0]), size=shape).astype(np.float32)
    zeros = rng.random(shape) < 0.1
    A[zeros] = 0.0
    return A


@pytest.mark.parametrize("trial", range(16))
def test_random_evict_rehydrate_rounds(trial):
    rng = np.random.default_rng(100 + trial)
    if trial % 2 == 0:
        tree_spec = ("full", int(rng.integers(2, 4)), int(rng.integers(2, 4)), int(rng.choice([40, 64, 96])))
    else:
        tree_spec = ("search", int(rng.integers(10, 30)), 3, 4, int(rng.choice([32, 72])))
    # half the trials in the 8-KV-head shape (nodes ≤ 128 slots, 16-slot pages): the fixed-layout
    # select_compact instantiation; the others take the runtime-layout kernel
    L, H, Hq = (1, 8, 32) if trial % 4 >= 2 else (2, 2, 8)
    preset = dict(tree=tree_spec, L=L, H=H, Hq=Hq, d=128, dtype="bf16", P=16, rho=0.3,
                  params=dict(l_tail=int(rng.choice([0, 2, 8])), k_min=int(rng.choice([0, 2]))),
                  active="highest_v")
    pr = Pair(preset, seed=trial)
    tree = pr.tree
    N = tree.num_nodes
    T = pr.ctx.score.shape[-1]
    A = _random_A(rng, (pr.ctx.L, pr.ctx.H, T))
    pr.ctx.score.copy_(torch.as_tensor(A))
    pr.ctx.arbor_invalidate_masses()
    leaves = synth.leaves_of(tree)
    k_now = [int(pr.orc.n[i]) for i in range(N)]
    for rnd in range(5):
        tree.active = [int(rng.choice(leaves))]
        # a random shrinking target: k ≤ k_cur, some nodes to 0, some unchanged
        k = []
        for i in range(N):
            kc = pr.orc.k_cur(i)
            r = rng.random()
            k.append(kc if r < 0.2 else (0 if r < 0.3 else int(rng.integers(0, kc + 1))))
        kd = torch.as_tensor(np.asarray(k, np.int32), device="cuda")
        ev = pr.ctx.arbor_evict(tree, kd, want_count=True)
        assert ev == pr.orc.evict(tree, k, A_f32=pr.gpu_A()), f"evicted count, round {rnd}"
        pr.check_kv_state()
        if rnd % 2 == 1:
            cand = [i for i in range(N) if pr.orc.k_cur(i) < pr.orc.n[i] and not tree.is_open[i]]
            if cand:
                pick = sorted(int(x) for x in rng.choice(cand, size=min(len(cand), 3), replace=False))
                pr.ctx.arbor_rehydrate(tree, pick)
                pr.orc.rehydrate(pick)
                pr.ctx.arbor_sync()
                pr.check_kv_state()
        k_now = [pr.orc.k_cur(i) for i in range(N)]
    assert sum(k_now) <= tree.total_tokens
