"""Phase timeline of the allocate kernel (a1 + a4) on C2 — needs a debug build:

    ARBOR_NVCC_FLAGS=-DARBOR_ALLOC_TRACE python -m paper_2605_22106_b200.build
    python profiles/alloc_trace.py

clock64() at the kernel's TRACE points (allocate.cu): 0 start, 1 geometry + weights done,
2 waterfill sums, 4/5 breakpoint search / active set, 6 done.  Prints cycle deltas (µs at
1.965 GHz), median over the two alternating leaves × 10 calls.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    import synth
    from paper_2605_22106_b200 import workload
    import paper_2605_22106_b200 as pk

    lib = pk.load_library()
    fn = lib.arbor_debug_set_alloc_trace
    fn.argtypes = [C.c_void_p, C.c_void_p]
    fn.restype = C.c_int32
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
    if cfg == "c3dpts":      # the DPTS loop's state (decode_step_prof.py c3dpts): 16 leaves
        T, D = 6, 8
        extra_nodes, extra_tokens, node_extra = workload.dpts_sizing(T, D)
        sc = workload.setup("c3", 0, extra_tokens=extra_tokens, extra_nodes=extra_nodes,
                            max_active=16, node_extra_tokens=node_extra)
        workload.warmup_leaf_cycling(sc, 1)
        run = workload.DptsRun(sc, n_active=16, transitions=T, swap=4, decode_steps=D, seed=0)
        for leaves_t in [run.base_leaves] + run.schedule:
            run.transition(leaves_t)
            for _ in range(D):
                run.decode()
        sets = [list(sc.tree.active)] * 2
    else:
        sc = workload.setup(cfg, 0)
        workload.warmup_leaf_cycling(sc, 1)
        sets = [[x] for x in sorted(synth.leaves_of(sc.tree), key=lambda x: -float(sc.tree.v[x]))[:2]]
    ctx, tree = sc.ctx, sc.tree
    tr = torch.zeros(16, dtype=torch.int64, device="cuda")
    assert fn(ctx._ctx, C.c_void_p(tr.data_ptr())) == 0
    s = torch.empty(tree.num_nodes, dtype=torch.float32, device="cuda")
    k = torch.empty(tree.num_nodes, dtype=torch.int32, device="cuda")
    B = sc.budget
    rows = []
    for i in range(20):
        tree.active = sets[i % 2]
        nA = len(tree.active)
        q = sc.queries(10_000 + i, nA)
        out = torch.empty_like(q)
        lse = torch.empty((nA, ctx.L, ctx.Hq), dtype=torch.float32, device="cuda")
        ctx.arbor_decode_step(tree, q, out, lse, s)
        tr.zero_()
        ctx.arbor_allocate(tree, s, B, k)
        torch.cuda.synchronize()
        rows.append(tr.cpu().numpy().copy())
    t = np.array(rows, dtype=np.float64)
    res = {}
    res["multisection_rounds"] = float(np.median(t[:, 7]))
    res["breakpoints"] = float(np.median(t[:, 8]))
    for j in (1, 2, 3, 4, 5, 6):
        ok = t[:, j] > 0
        if ok.any():
            res[f"t{j}_us"] = float(np.median((t[ok, j] - t[ok, 0]) / 1965.0))
    print(json.dumps({"config": cfg, "nodes": tree.num_nodes, "phase_end_us_from_start": res}))


if __name__ == "__main__":
    main()
