"""f1 measurement: the event-driven controller (Alg. 2) on an 8B-shaped Tree-of-Thoughts
search, 1 GPU — the Fig. 4-style peak-KV time series and the policy overhead
against decoding (the paper reports < 1.2 % of wall-clock).

Trace (seeded, synthetic): Llama-3.1-8B KV shape (32 layers × 8 KV × 32 Q heads, d 128,
bf16), a 128-token prompt, then `--expansions` ToT expansions (width 5, depth ≤ 4, chosen
∝ v): Transition to a new child, 128 decode steps into it (append K/V, tree decode attention
a9, score a2+a3, waterline check), Boundary at its close.  Two runs on the same trace:
  * FullKV: no controller (every token stays resident);
  * ArborKV: Controller with budget 𝓑 = ρ · (final FullKV tokens), δ = 128.
Device time per decode step and per policy event comes from CUDA events; retained tokens
and pages in use are sampled after every event and every 16 decode steps.
Usage (GPU box): python profiles/controller_trace.py --out profiles/r01_controller_trace.json
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(expansions, rho, t_node, seed, controlled, budget=None):
    import numpy as np
    import torch
    import synth
    from paper_2605_22106_b200 import workload

    dev = torch.device("cuda", 0)
    base = dict(workload.PRESETS["c2"], tree=("full", 1, 5, t_node))
    workload.PRESETS["ctl"] = base
    tree = synth.full_tree(1, 5, t_node, seed)
    extra = t_node * (expansions + 1)
    sc = workload.setup("ctl", seed, extra_tokens=extra, extra_nodes=expansions + 2,
                        profile=False, device=dev)
    ctx, tree = sc.ctx, sc.tree
    stream = torch.cuda.current_stream(dev)
    L, H, D = ctx.L, ctx.H, ctx.D
    rb = D * 2
    page_bytes = ctx.P * L * H * 2 * rb
    gen = torch.Generator(device=dev).manual_seed(seed + 99)
    final_tokens = t_node * (expansions + 1)
    B = budget if budget is not None else int(rho * final_tokens)
    ctl = workload.Controller(ctx, B, t_node) if controlled else None
    rng = np.random.default_rng(seed + 5)
    series, dec_ms, pol_ms, kinds = [], [], [], []
    tree.active = [0]
    step = [0]

    def timed(fn):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        return a, b

    def sample(tag):
        total = ctx.arbor_retained_tokens()
        pages = ctx.arbor_read_counters()[1]
        series.append({"step": step[0], "event": tag, "tokens": total,
                       "kv_GiB": pages * page_bytes / 2**30})

    def policy(kind, node=-1):
        if ctl is None:
            return
        fn = {"boundary": lambda: ctl.boundary(tree, node), "transition": lambda: ctl.transition(tree),
              "pressure": lambda: ctl.pressure(tree)}[kind]
        pol_ms.append(timed(fn))
        kinds.append(kind)
        sample(kind)

    def waterline():
        # Alg. 2 l.31-33 on the device: check + gated Pressure, no host sync (the device time
        # of every check counts as policy time, fired or not)
        if ctl is not None:
            pol_ms.append(timed(lambda: ctl.waterline_device(tree)))
            kinds.append("waterline")

    def decode():
        q = sc.queries(50_000 + step[0], 1)
        out = torch.empty_like(q)
        lse = torch.empty((1, L, ctx.Hq), dtype=torch.float32, device=dev)
        dec_ms.append(timed(lambda: ctx.arbor_decode_step(tree, q, out, lse)))
        step[0] += 1

    t0 = time.perf_counter()
    decode()
    policy("boundary", 0)
    sample("start")
    next_pos = t_node
    for _ in range(expansions):
        pick = synth.tot_expansion(tree, rng, 5, 4)
        if pick is None:
            break
        parent, v, u = pick
        child = tree.add_node(parent, next_pos, 0, True, v, u)
        ctx.arbor_open_node(child, next_pos)
        next_pos += t_node
        tree.active = [child]
        policy("transition")
        waterline()
        for t in range(t_node):
            k = torch.randn((L, H, 1, D), generator=gen, device=dev).to(torch.bfloat16)
            v_ = torch.randn((L, H, 1, D), generator=gen, device=dev).to(torch.bfloat16)
            ctx.arbor_append_kv(child, k, v_)
            tree.span_len[child] += 1
            decode()
            waterline()
            if t % 16 == 15:
                sample("decode")
        ctx.arbor_close_node(child)
        tree.is_open[child] = 0
        policy("boundary", child)
        waterline()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    dms = [a.elapsed_time(b) for a, b in dec_ms]
    pms = [a.elapsed_time(b) for a, b in pol_ms]
    rehyd = ctx.arbor_read_counters()[0]
    res = {"controlled": controlled, "budget": B if controlled else None, "rho": rho if controlled else 1.0,
           "nodes": tree.num_nodes, "final_tokens": int(tree.total_tokens),
           "decode_steps": len(dms), "decode_ms_total": sum(dms),
           "decode_ms_p50": statistics.median(dms),
           "policy_events": dict({k: kinds.count(k) for k in ("boundary", "transition", "waterline")},
                                 pressure_fired=ctx.arbor_pressure_events() if controlled else 0),
           "policy_ms_total": sum(pms), "policy_ms_p50_by_kind": {
               k: statistics.median([m for m, kk in zip(pms, kinds) if kk == k])
               for k in ("boundary", "transition", "waterline") if k in kinds},
           "policy_overhead_frac": sum(pms) / (sum(pms) + sum(dms)) if pms else 0.0,
           "rehydrations": rehyd,
           "peak_tokens": max(x["tokens"] for x in series),
           "peak_kv_GiB": max(x["kv_GiB"] for x in series),
           "final_kv_GiB": series[-1]["kv_GiB"], "host_wall_s": wall, "series": series}
    del sc, ctx
    torch.cuda.empty_cache()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--expansions", type=int, default=30)
    ap.add_argument("--t-node", type=int, default=128)
    ap.add_argument("--rho", type=float, default=0.3)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    full = run(a.expansions, 1.0, a.t_node, a.seed, controlled=False)
    arb = run(a.expansions, a.rho, a.t_node, a.seed, controlled=True)
    summary = {"workload": "f1 controller on an 8B-shaped ToT search (width 5, depth <= 4, "
                           f"{a.t_node}-token blocks, {a.expansions} expansions), 1 x B200",
               "fullkv": {k: v for k, v in full.items() if k != "series"},
               "arborkv": {k: v for k, v in arb.items() if k != "series"},
               "peak_kv_reduction": full["peak_kv_GiB"] / max(arb["peak_kv_GiB"], 1e-9),
               "series_fullkv": full["series"], "series_arborkv": arb["series"]}
    print(json.dumps({k: v for k, v in summary.items() if not k.startswith("series")}), flush=True)
    if a.out:
        with open(a.out, "w") as f:
            json.dump(summary, f, indent=1)


if __name__ == "__main__":
    main()
