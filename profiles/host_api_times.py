"""Host-side cost of each C-ABI call of the C2 step (the enqueue time; the device runs
behind).  python profiles/host_api_times.py"""
from __future__ import annotations

import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import synth
    from paper_2605_22106_b200 import workload
    from paper_2605_22106_b200.arbor import TreeArgs

    sc = workload.setup("c2", 0)
    ctx, tree = sc.ctx, sc.tree
    workload.warmup_leaf_cycling(sc, 1)
    leaves = sorted(synth.leaves_of(tree), key=lambda x: -float(tree.v[x]))[:2]
    trees = []
    for leaf in leaves:
        tree.active = [leaf]
        trees.append(TreeArgs.from_tree(tree))
    q = sc.queries(0, 1)
    out = torch.empty_like(q)
    lse = torch.empty((1, ctx.L, ctx.Hq), dtype=torch.float32, device="cuda")
    s = torch.empty(tree.num_nodes, dtype=torch.float32, device="cuda")
    k = torch.empty(tree.num_nodes, dtype=torch.int32, device="cuda")
    B = sc.budget
    ctx.arbor_save_state(0)
    snap = [t.clone() for t in (ctx.k_pool, ctx.v_pool, ctx.pos_pool, ctx.score)]
    T = {"decode_step": [], "allocate": [], "evict": []}
    for i in range(40):
        for dst, src in zip((ctx.k_pool, ctx.v_pool, ctx.pos_pool, ctx.score), snap):
            dst.copy_(src)
        ctx.arbor_load_state(0)
        torch.cuda.synchronize()
        ta = trees[i % 2]
        t0 = time.perf_counter(); ctx.arbor_decode_step(ta, q, out, lse, s)
        t1 = time.perf_counter(); ctx.arbor_allocate(ta, s, B, k)
        t2 = time.perf_counter(); ctx.arbor_evict(ta, k)
        t3 = time.perf_counter()
        torch.cuda.synchronize()
        if i >= 5:
            T["decode_step"].append((t1 - t0) * 1e6)
            T["allocate"].append((t2 - t1) * 1e6)
            T["evict"].append((t3 - t2) * 1e6)
    print(json.dumps({k2: round(statistics.median(v), 1) for k2, v in T.items()} | {"unit": "us host"}))


if __name__ == "__main__":
    main()
