"""Timeline of the select + compact kernel (a5+a6, evict.cu select_move_ws_kernel) on a B200.

Runs the bench's C2 (or C4 / C5) eviction step once with ARBOR_EVICT_TRACE=1 and reads the
globaltimer trace each warp writes (evict.cu EV_TRACE: 0 start after griddepcontrol.wait,
1 plan done, 2 first job handed (select) / started (move), 3 last job handed / done).  Prints
percentiles in µs relative to the earliest CTA start.  A diagnostic, not a bench.

    ARBOR_NVCC_FLAGS=-DARBOR_EVICT_TRACE_BUILD python -m paper_2605_22106_b200.build --force
    python profiles/evict_trace.py [c2|c4|c5] > gpurun_out/evict_trace_c2.json

(the timeline is compiled only into that diagnostic build; add -DARBOR_EVICT_PHASES for the
select-phase cycle sums)
"""
from __future__ import annotations

import ctypes as C
import json
import math
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

    cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
    sc = workload.setup(cfg, 0)
    workload.warmup_leaf_cycling(sc)
    tree, ctx = sc.tree, sc.ctx
    tree.active = [synth.highest_v_leaf(tree)]
    s = torch.empty(tree.num_nodes, dtype=torch.float32, device="cuda")
    q = sc.queries(10 ** 6, 1)
    out = torch.empty_like(q)
    lse = torch.empty((1, ctx.L, ctx.Hq), dtype=torch.float32, device="cuda")
    ctx.arbor_decode_step(tree, q, out, lse, s)
    k = torch.empty(tree.num_nodes, dtype=torch.int32, device="cuda")
    ctx.arbor_allocate(tree, s, sc.budget, k)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    flush.zero_()
    torch.cuda.synchronize()
    os.environ["ARBOR_EVICT_TRACE"] = "1"
    ctx.arbor_evict(tree, k)
    torch.cuda.synchronize()
    del os.environ["ARBOR_EVICT_TRACE"]
    lib = pk.load_library()
    ctas = torch.cuda.get_device_properties(0).multi_processor_count * 2
    n = ctas * 16 * 16
    buf = (C.c_longlong * n)()
    lib.arbor_debug_evict_trace.argtypes = [C.POINTER(C.c_longlong), C.c_longlong]
    assert lib.arbor_debug_evict_trace(buf, n) == 0
    tr = np.frombuffer(buf, dtype=np.int64).reshape(ctas, 16, 16).astype(np.float64)
    t0 = tr[:, :, 0][tr[:, :, 0] > 0].min()
    rel = (tr - t0) / 1e3
    valid = tr > 0

    def pct(x):
        x = x[np.isfinite(x)]
        return [round(float(v), 2) for v in np.percentile(x, [0, 10, 50, 90, 100])] if x.size else None

    sel, mov = slice(0, 8), slice(8, 16)
    res = {
        "config": cfg,
        "ctas": ctas,
        "pct": "min/p10/p50/p90/max µs after the first CTA start",
        "cta_start": pct(np.where(valid[:, 0, 0], rel[:, 0, 0], np.nan)),
        "plan_loads_done": pct(np.where(valid[:, 0, 4], rel[:, 0, 4], np.nan)),
        "plan_scans_done": pct(np.where(valid[:, 0, 5], rel[:, 0, 5], np.nan)),
        "plan_done": pct(np.where(valid[:, 0, 1], rel[:, 0, 1], np.nan)),
        "select_first_rank_start": pct(np.where(valid[:, sel, 6], rel[:, sel, 6], np.nan).ravel()),
        "select_first_job": pct(np.where(valid[:, sel, 2], rel[:, sel, 2], np.nan).ravel()),
        "move_first_job": pct(np.where(valid[:, mov, 2], rel[:, mov, 2], np.nan).ravel()),
        "select_done": pct(np.where(valid[:, sel, 3], rel[:, sel, 3], np.nan).ravel()),
        "move_done": pct(np.where(valid[:, mov, 3], rel[:, mov, 3], np.nan).ravel()),
    }
    # move warps: SM id, jobs, rows (slot 7) against their finishing time
    info = tr[:, mov, 7].astype(np.int64)
    smid, jobs, rows = info >> 40, (info >> 20) & 0xFFFFF, info & 0xFFFFF
    done = rel[:, mov, 3]
    ok = valid[:, mov, 3]
    res["move_jobs"] = pct(np.where(ok, jobs, np.nan).ravel())
    res["move_rows"] = pct(np.where(ok, rows, np.nan).ravel())
    # cycles → µs at 1.965 GHz: move warps waiting for a job, select warps waiting for a slot
    res["move_wait_full_us"] = pct(np.where(ok, tr[:, mov, 6] / 1965.0, np.nan).ravel())
    res["select_wait_empty_us"] = pct(np.where(valid[:, sel, 3], tr[:, sel, 7] / 1965.0, np.nan).ravel())
    if (tr[:, sel, 8:14] > 0).any():   # -DARBOR_EVICT_PHASES builds: select-phase µs per warp
        names = ["issue_next", "keys", "threshold", "lists", "handoff", "data_wait"]
        okk = valid[:, sel, 3]
        res["select_phase_us"] = {nm: pct(np.where(okk, tr[:, sel, 8 + i] / 1965.0, np.nan).ravel())
                                  for i, nm in enumerate(names)}
        res["select_items"] = pct(np.where(okk, tr[:, sel, 14], np.nan).ravel())
    late = np.argsort(np.where(ok, done, -1).ravel())[::-1][:12]
    res["latest_moves"] = [{"cta": int(i // 8), "sm": int(smid.ravel()[i]), "jobs": int(jobs.ravel()[i]),
                            "rows": int(rows.ravel()[i]), "done": round(float(done.ravel()[i]), 2)}
                           for i in late]
    # per SM: rows moved by its move warps and the time its last one finished
    sm_rows, sm_done = {}, {}
    for c in range(ctas):
        for w in range(8):
            if not ok[c, w]:
                continue
            m = int(smid[c, w])
            sm_rows[m] = sm_rows.get(m, 0) + int(rows[c, w])
            sm_done[m] = max(sm_done.get(m, 0.0), float(done[c, w]))
    ms = sorted(sm_done, key=lambda m: sm_done[m])
    res["sm_rows_vs_done"] = [[m, sm_rows[m], round(sm_done[m], 2)] for m in ms[:5] + ms[-8:]]
    if len(ms) > 2:
        res["corr_rows_done_per_sm"] = float(np.corrcoef([sm_rows[m] for m in ms], [sm_done[m] for m in ms])[0, 1])
        res["corr_smid_done"] = float(np.corrcoef(ms, [sm_done[m] for m in ms])[0, 1])
    print(json.dumps(res))


if __name__ == "__main__":
    main()
