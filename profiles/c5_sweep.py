"""configs[4]: budget sweep on 8B-shaped search trees, 1 GPU.

For every tree size N ∈ {64, 128, 256, 512} (search_tree(N, 3, 8, 128): 8k … 64k cached
tokens) and budget ratio ρ ∈ {0.125, 0.25, 0.5, 1.0}, from the same full-retention state:
  * the eviction step (a9 → a2+a3 → a1+a4 → a5+a6, the bench.py step) on the device:
    eviction tokens/s = cached tokens ÷ step time (CUDA events, median of `--reps`);
  * peak KV after the step: pages in use × page bytes, against full retention;
  * a decode step on the evicted state (a9 + a2/a3 for the active leaf): tokens/s against
    ρ = 1.0 — the eviction's effect on decode (paper: < 1.2 % policy overhead);
  * infeasible budgets (B < Σ pinned n + Σ floors) are reported with `min_feasible`.
Prints one JSON object per (N, ρ) and a summary list; writes profiles/r01_c5_sweep.json
with --out.  Run on a GPU box: python profiles/c5_sweep.py --out profiles/r01_c5_sweep.json
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import synth
    from paper_2605_22106_b200 import workload
    from paper_2605_22106_b200.arbor import ArborError, TreeArgs

    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="64,128,256,512")
    ap.add_argument("--rhos", default="0.125,0.25,0.5,1.0")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream(dev)
    base = workload.PRESETS["c5"]
    results = []
    for N in [int(x) for x in args.sizes.split(",")]:
        workload.PRESETS["c5_sweep"] = dict(base, tree=("search", N, 3, 8, 128))
        sc = workload.setup("c5_sweep", args.seed, profile=True, device=dev)
        ctx, tree = sc.ctx, sc.tree
        workload.warmup_leaf_cycling(sc)
        leaf = synth.highest_v_leaf(tree)
        tree.active = [leaf]
        ta = TreeArgs.from_tree(tree)
        T = tree.total_tokens
        q = sc.queries(10_000, 1)
        out = torch.empty_like(q)
        lse = torch.empty((1, ctx.L, ctx.Hq), dtype=torch.float32, device=dev)
        s_buf = torch.empty(tree.num_nodes, dtype=torch.float32, device=dev)
        k_buf = torch.empty(tree.num_nodes, dtype=torch.int32, device=dev)
        snap = [ctx.k_pool.clone(), ctx.v_pool.clone(), ctx.pos_pool.clone(), ctx.score.clone()]
        ctx.arbor_save_state(0)
        ctx.arbor_set_profiling(False)
        rb = ctx.D * (2 if base["dtype"] == "bf16" else 4)
        page_bytes = ctx.P * ctx.L * ctx.H * 2 * rb
        full_pages = ctx.arbor_read_counters()[1]

        def restore():
            ctx.k_pool.copy_(snap[0])
            ctx.v_pool.copy_(snap[1])
            ctx.pos_pool.copy_(snap[2])
            ctx.score.copy_(snap[3])
            ctx.arbor_load_state(0)

        def timed(fn, reps):
            ms = []
            for _ in range(reps):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                fn()
                b.record(stream)
                b.synchronize()
                ms.append(a.elapsed_time(b))
            return statistics.median(ms)

        decode_full = None
        for rho in [float(x) for x in args.rhos.split(",")]:
            B = int(math.floor(rho * T))
            rec = {"N": N, "tokens": T, "rho": rho, "budget": B}
            restore()
            try:
                ctx.arbor_decode_step(ta, q, out, lse, s_buf)
                ctx.arbor_allocate(ta, s_buf, B, k_buf)
            except ArborError as e:
                if e.status != 3:
                    raise
                ctx.arbor_sync()
                rec.update(infeasible=True, min_feasible=e.min_feasible)
                results.append(rec)
                print(json.dumps(rec), flush=True)
                continue

            step_ms = []
            for r in range(args.reps + 3):
                restore()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                ctx.arbor_decode_step(ta, q, out, lse, s_buf)
                ctx.arbor_allocate(ta, s_buf, B, k_buf)
                ctx.arbor_evict(ta, k_buf)
                b.record(stream)
                b.synchronize()
                if r >= 3:
                    step_ms.append(a.elapsed_time(b))
            kept = sum(int(x) for x in k_buf.cpu().tolist())
            pages = ctx.arbor_read_counters()[1]

            def decode():
                ctx.arbor_decode_step(ta, q, out, lse, s_buf)

            dms = timed(decode, args.reps)
            if rho == 1.0:
                decode_full = dms
            ms = statistics.median(step_ms)
            rec.update(infeasible=False, step_ms=ms, eviction_tokens_per_s=T / (ms / 1e3),
                       kept_tokens=kept, pages_in_use=pages, full_pages=full_pages,
                       peak_kv_GiB=pages * page_bytes / 2**30,
                       full_kv_GiB=full_pages * page_bytes / 2**30,
                       kv_reduction=full_pages / max(pages, 1), decode_step_ms=dms,
                       decode_tokens_per_s=1 / (dms / 1e3))
            results.append(rec)
            print(json.dumps(rec), flush=True)
        for rec in results:
            if rec["N"] == N and not rec.get("infeasible") and decode_full:
                rec["decode_vs_full_retention"] = decode_full / rec["decode_step_ms"]
        del sc, ctx, snap
        torch.cuda.empty_cache()
    summary = {"workload": "C5 budget sweep (configs[4]): search_tree(N, 3, 8, 128), Llama-3.1-8B "
                           "KV shape (32 L x 8 KV x 32 Q heads, d 128, bf16), 1 x B200",
               "results": results}
    print(json.dumps(summary), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(summary, f, indent=1)


if __name__ == "__main__":
    main()
