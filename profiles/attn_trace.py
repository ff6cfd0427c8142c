"""Per-tile timeline of the tensor-core tree decode attention (a9, attn_tc.cu) on a B200.

Runs the C2 (1 leaf) or C3 (16 leaves) decode step with ARBOR_TC_TRACE=1, reads the clock64
trace the kernel writes (event ids in attn_tc.cu: 0 producer turn, 1 stage free, 2 TMA
issued, 3 MMA1 issued, 12 S ready, 5 MMA2 issued, 13 O ready, 7 softmax saw data, 8 softmax
saw S, 9 P written, 10 epilogue saw O, 11 partials stored) and prints per-event medians
relative to the producer turn plus the CTA span.  Trace mode serialises the MMA issuer on
its own commits, so absolute spans are upper bounds; it is a diagnostic, not a bench.

    ARBOR_NVCC_FLAGS=-DARBOR_TC_TRACE_BUILD python -m paper_2605_22106_b200.build --force
    python profiles/attn_trace.py [c2|c3] > gpurun_out/attn_trace_c2.json

(the trace is compiled only into that diagnostic build)
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
    from paper_2605_22106_b200 import workload
    import paper_2605_22106_b200 as pk

    cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
    if cfg == "c3dpts":      # the DPTS loop's state: a few transitions, open children decoding
        T, D = 6, 8
        extra_nodes, extra_tokens, node_extra = workload.dpts_sizing(T, D)
        sc = workload.setup("c3", 0, extra_tokens=extra_tokens, extra_nodes=extra_nodes,
                            max_active=16, node_extra_tokens=node_extra)
        workload.warmup_leaf_cycling(sc, 1)
        run = workload.DptsRun(sc, n_active=16, transitions=T, swap=4, decode_steps=D, seed=0)
        for leaves in [run.base_leaves] + run.schedule:
            run.transition(leaves)
            for _ in range(D):
                run.decode()
        for ch in sc.tree.active:
            run._append(ch)
    else:
        sc = workload.setup(cfg, 0)
    tree = sc.tree
    nA = len(tree.active)
    q = sc.queries(0, nA)
    out = torch.empty_like(q)
    lse = torch.empty((nA, sc.ctx.L, sc.ctx.Hq), dtype=torch.float32, device=q.device)
    for _ in range(3):
        sc.ctx.arbor_tree_decode_attn(tree, q, out, lse)
    torch.cuda.synchronize()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=q.device)
    if os.environ.get("TRACE_COLD"):
        flush.zero_()                      # L2 flush: K/V come from HBM
        torch.cuda.synchronize()
    os.environ["ARBOR_TC_TRACE"] = "1"
    sc.ctx.arbor_tree_decode_attn(tree, q, out, lse)
    torch.cuda.synchronize()
    del os.environ["ARBOR_TC_TRACE"]
    lib = pk.load_library()
    n = 148 * 64 * 16
    buf = (C.c_longlong * n)()
    lib.arbor_debug_tc_trace.argtypes = [C.POINTER(C.c_longlong), C.c_longlong]
    assert lib.arbor_debug_tc_trace(buf, n) == 0
    tr = np.frombuffer(buf, dtype=np.int64).reshape(148, 64, 16)
    clk_ghz = 1.965
    spans_ns = [(tr[c, 63, 1] - tr[c, 63, 0]) for c in range(148) if tr[c, 63, 1] > 0]
    ev = {}
    tiles_per_cta = []
    for c in range(148):
        k = 0
        while k < 63 and (tr[c, k, 11] > 0 or tr[c, k, 0] > 0):
            k += 1
        tiles_per_cta.append(k)
        for t in range(k):
            for e in (1, 2, 3, 12, 5, 13, 7, 8, 9, 10, 11):
                if tr[c, t, e] > 0:
                    ev.setdefault(e, []).append((tr[c, t, e] - tr[c, t, 0]) / clk_ghz / 1000.0)
    # per-tile completion spacing (epilogue done of tile k+1 − tile k)
    gaps = []
    firsts = []
    for c in range(148):
        k = tiles_per_cta[c]
        if k:
            firsts.append(tr[c, 0, 11] / clk_ghz / 1000.0)
        for t in range(1, k):
            gaps.append((tr[c, t, 11] - tr[c, t - 1, 11]) / clk_ghz / 1000.0)
    starts = [tr[c, 63, 0] for c in range(148) if tr[c, 63, 0] > 0]
    t0 = min(starts)
    res = {
        "config": cfg, "active_leaves": nA, "cold_l2": bool(os.environ.get("TRACE_COLD")),
        "tiles_total_est": int(sum(tiles_per_cta)),
        "cta_span_us_p50_max": [float(np.median(spans_ns)) / 1e3, float(np.max(spans_ns)) / 1e3],
        "cta_start_skew_us_max": float(max(starts) - t0) / 1e3,
        "cta_end_us_max": float(max(tr[c, 63, 1] for c in range(148)) - t0) / 1e3,
        "tiles_per_cta_min_max": [int(min(tiles_per_cta)), int(max(tiles_per_cta))],
        "first_tile_done_us_p50": float(np.median(firsts)),
        "tile_gap_us_p10_p50_p90": [float(x) for x in np.percentile(gaps, [10, 50, 90])] if gaps else None,
        "event_us_after_producer_turn_p50": {str(e): float(np.median(v)) for e, v in sorted(ev.items())},
    }
    print(json.dumps(res))


if __name__ == "__main__":
    main()
