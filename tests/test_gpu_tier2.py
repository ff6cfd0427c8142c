"""Tier (ii) end-to-end discrete parity (SURVEY §8(c) "What bit-exact is tested against").

The oracle computes A and s ITSELF (fp64 scores of its own decode), allocates and evicts;
the GPU runs the same seeded steps through the C ABI.  Budgets k and kept sets must agree,
and every discrete difference must carry a tie certificate:
  * k: some node's f32 s differs between the two sides (the float tier allows 1e-5) and the
    oracle fed the GPU's own s (tier (i)) reproduces the GPU's k exactly;
  * kept set of a (row, node) with equal k: each swapped pair (x kept only on the GPU,
    y kept only by the oracle, matched in key order) has an oracle key gap A(y) − A(x) no
    larger than the two sides' combined A error at x and y (the keys are within float
    error of a tie, so either order is correct).
Observed difference counts are printed (evidence, not a tolerance).
"""
import math

import numpy as np
import pytest
import torch

from paper_2605_22106_b200 import workload

from gpu_helpers import Pair

pytestmark = pytest.mark.gpu

MID = dict(tree=("full", 4, 4, 96), L=2, H=4, Hq=16, d=128, dtype="bf16", P=16, rho=0.25,
           params={}, active="highest_v")


def _kept_sets(pr, node):
    kc, pages, pos, _, _, _ = pr.gpu_node(node)
    return kc, pos


@pytest.mark.parametrize("preset,seed,steps", [("c1", 0, 4), ("c1", 1, 4), ("mid", 2, 2)])
def test_end_to_end_discrete_parity_with_tie_certificates(preset, seed, steps):
    p = workload.PRESETS["c1"] if preset == "c1" else MID
    pr = Pair(p, seed)
    pr.warmup(steps_per_leaf=steps, check=False)
    pr.decode_both(check=True)
    sc = pr.ctx.arbor_read_scores(pr.tree.num_nodes)
    s_gpu = [float(x) for x in sc["s"]]
    _, s_ref = pr.orc.msve(pr.tree)                     # the oracle's own fp64 → f32 s
    B = int(math.floor(p["rho"] * pr.tree.total_tokens)) if preset != "c1" else 112
    k = torch.empty(pr.tree.num_nodes, dtype=torch.int32, device="cuda")
    pr.ctx.arbor_allocate(pr.tree, torch.as_tensor(np.array(s_gpu, np.float32), device="cuda"), B, k)
    k_gpu = k.cpu().tolist()
    k_ref = pr.orc.allocate(pr.tree, s_ref, B)
    n_s_diff = sum(1 for a, b in zip(s_gpu, s_ref) if np.float32(a) != np.float32(b))
    for a, b in zip(s_gpu, s_ref):
        assert abs(a - b) <= 1e-5 * abs(b)
    if k_gpu != k_ref:
        assert n_s_diff > 0, "k differs although s is identical on both sides"
        st, k_i, _ = pr.discrete_allocate(s_gpu, B)
        assert st == 0 and k_i == k_gpu, "the GPU's k is not the oracle's allocation of the GPU's s"
    A_gpu = pr.gpu_A()[:, :, :pr.orc.Tmax].astype(np.float64)
    A_ref = pr.orc.A
    # evict on both sides: the GPU with its k, the oracle with its own k and its own A (f32)
    pr.ctx.arbor_evict(pr.tree, k)
    before = {i: pr.orc.kept[i].copy() for i in range(pr.tree.num_nodes)}
    pr.orc.evict(pr.tree, k_ref)
    n_rows = n_rows_diff = n_pairs = 0
    for i in range(pr.tree.num_nodes):
        kc, pos = _kept_sets(pr, i)
        if kc != pr.orc.k_cur(i):
            assert k_gpu[i] != k_ref[i]                    # certified at the k level above
            continue
        a0 = int(pr.tree.span_start[i])
        for l in range(pr.ctx.L):
            for h in range(pr.ctx.H):
                n_rows += 1
                g = set(int(x) for x in pos[l, h])
                r = set(int(x) for x in pr.orc.kept[i][l, h])
                if g == r:
                    continue
                n_rows_diff += 1
                xs = sorted(g - r, key=lambda t: (A_ref[l, h, a0 + t], t))
                ys = sorted(r - g, key=lambda t: (A_ref[l, h, a0 + t], t))
                assert len(xs) == len(ys)
                for x, y in zip(xs, ys):
                    n_pairs += 1
                    gap = abs(A_ref[l, h, a0 + y] - A_ref[l, h, a0 + x])
                    err = (abs(A_gpu[l, h, a0 + x] - A_ref[l, h, a0 + x]) +
                           abs(A_gpu[l, h, a0 + y] - A_ref[l, h, a0 + y]))
                    # f32 rounding of the oracle's keys counts as error too
                    err += 2 ** -23 * (abs(A_ref[l, h, a0 + x]) + abs(A_ref[l, h, a0 + y]))
                    assert gap <= err, (i, l, h, x, y, gap, err)
    print(f"tier (ii) {preset} seed {seed}: s differs on {n_s_diff} nodes, k equal: "
          f"{k_gpu == k_ref}, kept sets differ on {n_rows_diff}/{n_rows} rows "
          f"({n_pairs} certified swaps)")
