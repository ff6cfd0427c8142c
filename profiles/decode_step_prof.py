"""Decode-step driver for ncu / timing: N arbor_decode_step calls on a preset (c2: 1 leaf,
c3: 16 DPTS leaves on the same 8B-shaped tree), full retention, device-resident inputs.

    python profiles/decode_step_prof.py c3 [steps]        # prints per-call CUDA-event µs
    POST_TRACE=1 … (decode_post phase timeline: a -DARBOR_POST_TRACE_BUILD build)
    ncu -k regex:"attn_tc|decode_post" ... python profiles/decode_step_prof.py c3 3
"""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2605_22106_b200 import workload

    cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    if cfg == "c3dpts":      # the DPTS loop's state: a few transitions, open children decoding
        T, D = 6, 8
        extra_nodes, extra_tokens, node_extra = workload.dpts_sizing(T, D)
        sc = workload.setup("c3", 0, profile=True, extra_tokens=extra_tokens,
                            extra_nodes=extra_nodes, max_active=16, node_extra_tokens=node_extra)
        workload.warmup_leaf_cycling(sc, 1)
        run = workload.DptsRun(sc, n_active=16, transitions=T, swap=4, decode_steps=D, seed=0)
        for leaves in [run.base_leaves] + run.schedule:
            run.transition(leaves)
            for _ in range(D):
                run.decode()
    else:
        sc = workload.setup(cfg, 0, profile=True)
    ctx, tree = sc.ctx, sc.tree
    nA = len(tree.active)
    qs = [sc.queries(i, nA) for i in range(2)]
    out = torch.empty_like(qs[0])
    lse = torch.empty((nA, ctx.L, ctx.Hq), dtype=torch.float32, device=qs[0].device)
    s = torch.empty(tree.num_nodes, dtype=torch.float32, device=qs[0].device)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=qs[0].device)
    for i in range(3):
        ctx.arbor_decode_step(tree, qs[i % 2], out, lse, s)
    torch.cuda.synchronize()
    ctx.arbor_set_profiling(True)
    ctx.arbor_reset_stage_times()
    ts = []
    for i in range(steps):
        flush.zero_()                                   # L2 flush between steps
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ctx.arbor_decode_step(tree, qs[i % 2], out, lse, s)
        e1.record()
        ts.append((e0, e1))
    torch.cuda.synchronize()
    st = ctx.arbor_stage_times()
    ctx.arbor_set_profiling(False)
    us = sorted(a.elapsed_time(b) * 1e3 for a, b in ts)
    res = {"config": cfg, "active_leaves": nA, "decode_step_us_p50": us[len(us) // 2],
           "stage_us": {k: round(v * 1e3, 2) for k, v in st.items() if v}}
    if os.environ.get("POST_TRACE"):
        # one more step with the decode_post phase trace (score.cu POST_TRACE): percentiles
        # over CTAs of each phase end, µs after the earliest CTA start
        import ctypes as C
        import numpy as np
        import paper_2605_22106_b200 as pk
        os.environ["ARBOR_POST_TRACE"] = "1"
        flush.zero_()
        ctx.arbor_decode_step(tree, qs[0], out, lse, s)
        torch.cuda.synchronize()
        del os.environ["ARBOR_POST_TRACE"]
        lib = pk.load_library()
        n = ctx.L * ctx.H * 64 * 16
        buf = (C.c_longlong * n)()
        lib.arbor_debug_post_trace.argtypes = [C.POINTER(C.c_longlong), C.c_longlong]
        assert lib.arbor_debug_post_trace(buf, n) == 0
        tr = np.frombuffer(buf, dtype=np.int64).reshape(-1, 16).astype(np.float64)
        tr = tr[tr[:, 0] > 0]
        t0 = tr[:, 0].min()
        names = ["start", "pdl_wait", "a_lse", "b_out", "score_A", "row_ticket", "masses",
                 "ticket", "last_msve"]
        ph = {}
        for e, nm in enumerate(names):
            x = tr[:, e]
            x = (x[x > 0] - t0) / 1e3
            if x.size:
                ph[nm] = [round(float(v), 2) for v in np.percentile(x, [0, 50, 90, 100])]
        res["post_trace_us_min_p50_p90_max"] = ph
        res["post_ctas"] = int(tr.shape[0])
    print(json.dumps(res))


if __name__ == "__main__":
    main()
