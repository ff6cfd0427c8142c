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
    sc = workload.setup(cfg, 0)
    ctx, tree = sc.ctx, sc.tree
    workload.warmup_leaf_cycling(sc, 1)
    tr = torch.zeros(16, dtype=torch.int64, device="cuda")
    assert fn(ctx._ctx, C.c_void_p(tr.data_ptr())) == 0
    leaves = sorted(synth.leaves_of(tree), key=lambda x: -float(tree.v[x]))[:2]
    s = torch.empty(tree.num_nodes, dtype=torch.float32, device="cuda")
    k = torch.empty(tree.num_nodes, dtype=torch.int32, device="cuda")
    B = sc.budget
    rows = []
    for i in range(20):
        tree.active = [leaves[i % 2]]
        q = sc.queries(10_000 + i, 1)
        out = torch.empty_like(q)
        lse = torch.empty((1, ctx.L, ctx.Hq), dtype=torch.float32, device="cuda")
        ctx.arbor_decode_step(tree, q, out, lse, s)
        tr.zero_()
        ctx.arbor_allocate(tree, s, B, k)
        torch.cuda.synchronize()
        rows.append(tr.cpu().numpy().copy())
    t = np.array(rows, dtype=np.float64)
    res = {}
    for j in (1, 2, 4, 5, 6):
        ok = t[:, j] > 0
        if ok.any():
            res[f"t{j}_us"] = float(np.median((t[ok, j] - t[ok, 0]) / 1965.0))
    print(json.dumps({"config": cfg, "nodes": tree.num_nodes, "phase_end_us_from_start": res}))


if __name__ == "__main__":
    main()
