#!/usr/bin/env python
"""ArborKV per-step KV-eviction benchmark on B200 (BASELINE.json metric).

A step is one pass of the whole hot path over the workload:
  a9 tree decode attention (→ LSE) → a2 score accumulation → a3 node mass + MSVE
  (→ a10 NCCL all-reduce when N > 1) → a1 geometry (the active leaf changes every step) →
  a4 TAE allocation → a5+a6 select + compact,
on configs[1] (C2: Llama-3.1-8B-shaped KV, ToT depth 4 × width 5, 19,968 cached tokens,
ρ = 0.25) by default.  Each step starts from the same full-retention state (restored
outside the timed region with device copies of the pools, A and the library state), so
`value` = cached tokens evicted-over per second of device time.  Rehydration (a7/a8,
PCIe-bound) is measured separately and reported under "rehydrate".

  python bench.py [--gpus N --steps K --warmup W --config c2 --impl arbor|reference]
Multi-GPU: launched by torchrun, one rank per GPU, KV heads sharded across ranks.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "eviction tokens/s; tree decode-attn HBM GB/s vs ~8 TB/s peak; 1/2/4/8 GPUs"
NOMINAL_HBM = 8000.0


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


# ---------------------------------------------------------------- clocks sampler
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = max(smax, float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------- distributed
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def run_reference(args):
    """--impl reference: the CPU oracle (oracle/), as it stands, on the host cores (one
    worker process per core over layers), on the same workload, inputs, warm-up and step
    as the GPU arm; same metric.  Under torchrun only rank 0 runs it."""
    ws, rank, _ = dist_env()
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo", init_method="env://")
        if rank != 0:
            dist.barrier()
            return
    if args.config == "c3":
        print(json.dumps({"impl": "reference", "unavailable": "the reference arm covers the bulk "
                          "eviction configs (c2, c4, c5); c3 is a transition loop"}), flush=True)
        return
    import torch
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    K, V, q_warm, q_step, order, leaves, B = bench_inputs(args.config, args.seed, dev)
    res = oracle_host_run(args.config, args.seed, args.warmup, args.steps, K, V, q_warm, q_step,
                          order, leaves, B, target_s=150.0)
    line = {"impl": "reference", "metric": METRIC, "value": res["value"], "unit": "tokens/s",
            "n_gpus": args.gpus, "steps": res["steps_timed"], "warmup": args.warmup,
            "ms_per_step": res["ms_per_step"], "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic" + ("" if dev == "cuda" else
                                                                        " (CPU generator)"),
            "config": workload_config(args.config, 1),
            "cpu_baseline": {"value": res["value"], "unit": "tokens/s", "cores": res["cores"],
                             "kind": "oracle", "sample": res["sample"],
                             "cpu_model": res["cpu_model"],
                             "single_thread_equiv_tokens_per_s": res["single_thread_equiv_tokens_per_s"],
                             "wall_s": res["wall_s"]},
            "e2e": {"value": res["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def workload_config(name, ws):
    from paper_2605_22106_b200.workload import PRESETS
    p = PRESETS[name]
    t = p["tree"]
    desc = {"c1": "C1 tiny tree (configs[0])", "c2": "C2 Llama-3.1-8B-shaped ToT depth4 x width5 (configs[1])",
            "c3": "C3 DPTS frontier 16 branches (configs[2])",
            "c4": "C4 Qwen2.5-32B-shaped deep tree (configs[3])",
            "c5": "C5 8B-shaped 64k-token tree (configs[4])"}[name]
    return {"workload": desc, "tree": f"{t[0]}_tree{tuple(t[1:])}", "layers": p["L"],
            "kv_heads": p["H"], "q_heads": p["Hq"], "head_dim": p["d"], "kv_dtype": p["dtype"],
            "page_size": p["P"], "rho": p["rho"],
            "parallelism": f"kv-head shards x{ws}" if ws > 1 else "single GPU",
            "l2": ("inputs > L2 (KV pools >> 126 MB); between steps a pool-restore copy, then "
                   "(c2/c4/c5) a 256 MB read pass that flushes L2 of its dirty lines"
                   if name != "c3" else "inputs > L2 (KV pools >> 126 MB)")}


# ---------------------------------------------------------------- CPU oracle on the host cores
_FLEET = {}          # set before the workers fork (copy-on-write inputs)


def _cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def _fleet_worker(conn, l0, l1):
    """One host core: the oracle (as it stands) over layers [l0, l1) — all KV heads of them.
    Commands: warm-up (the GPU arm's leaf-cycling warm-up, same queries), snapshot, step
    (restore → decode attention → score), evict (with the parent's k)."""
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(limits=1)
    except ImportError:
        pass
    import copy
    from oracle.state import ArborOracle
    F = _FLEET
    tree, p = F["tree"], F["preset"]
    o = ArborOracle(F["K"][l0:l1].double().numpy(), F["V"][l0:l1].double().numpy(), p["Hq"],
                    p["P"], F["num_pages"], F["params"], num_layers_global=p["L"],
                    num_q_heads_global=p["Hq"])
    for i in range(tree.num_nodes):
        o.open_node(i, int(tree.span_start[i]))
        o.append(i, int(tree.span_len[i]))
        o.close_node(i)
    state_keys = ("kept", "pages", "free", "A", "Nq", "Mclose", "s_last", "rehydrations")
    snap = None

    def q_of(qs, j):
        return qs[j][:, l0:l1].double().numpy()

    conn.send("ready")
    while True:
        cmd = conn.recv()
        t0 = time.perf_counter()
        if cmd[0] == "warm":
            for j, leaf in enumerate(cmd[1]):
                tree.active = [leaf]
                o.score_accumulate(tree, q_of(F["q_warm"], j))
            conn.send(time.perf_counter() - t0)
        elif cmd[0] == "snap":
            snap = {k: copy.deepcopy(getattr(o, k)) for k in state_keys}
            conn.send(0.0)
        elif cmd[0] == "step":
            for k_, v_ in snap.items():
                setattr(o, k_, copy.deepcopy(v_))
            tree.active = [cmd[1]]
            q = q_of(F["q_step"], cmd[2])
            _, lse = o.decode(tree, q)
            o.score_accumulate(tree, q, lse)
            masses = o.masses()
            conn.send((time.perf_counter() - t0, masses, list(o.Nq), list(o.Mclose)))
        elif cmd[0] == "evict":
            tree.active = [cmd[1]]
            ev = o.evict(tree, cmd[2])
            conn.send((time.perf_counter() - t0, ev))
        else:
            conn.send(None)
            return


class OracleFleet:
    """The CPU oracle (oracle/, as it stands, unmodified and untuned) on the host cores:
    one forked worker process per core, each owning a contiguous range of layers (every KV
    head of them, numpy/BLAS limited to one thread), running the rows' work (decode
    attention, score, node masses, select + compact); the node-level work (MSVE from the
    summed exact integer masses, TAE allocation) runs once, in the parent.  Same inputs as
    the GPU arm (its K/V and queries), the same leaf-cycling warm-up, the same step."""

    def __init__(self, config, seed, K, V, q_warm, q_step, cores=None):
        import multiprocessing as mp
        from oracle.state import default_params
        from paper_2605_22106_b200 import workload
        p = workload.PRESETS[config]
        self.preset, self.config = p, config
        self.tree = workload.build_tree(p, seed)
        self.params = default_params(**p["params"])
        L = p["L"]
        self.cores = max(1, min(cores or _host_cores(), L))
        bounds = [round(i * L / self.cores) for i in range(self.cores + 1)]
        _FLEET.update(tree=self.tree, preset=p, K=K, V=V, q_warm=q_warm, q_step=q_step,
                      params=self.params,
                      num_pages=sum(-(-int(x) // p["P"]) for x in self.tree.span_len) + 64)
        ctx = mp.get_context("fork")
        self.conns, self.procs = [], []
        for w in range(self.cores):
            a, b = ctx.Pipe()
            pr = ctx.Process(target=_fleet_worker, args=(b, bounds[w], bounds[w + 1]), daemon=True)
            pr.start()
            self.conns.append(a)
            self.procs.append(pr)
        for c in self.conns:
            assert c.recv() == "ready"

    def _all(self, msg):
        for c in self.conns:
            c.send(msg)
        return [c.recv() for c in self.conns]

    def warmup(self, order):
        return max(self._all(("warm", order)))

    def snapshot(self):
        self._all(("snap",))

    def step(self, leaf, qi, budget):
        """One timed step (wall clock of the parent, IPC included); returns (seconds,
        single-thread-equivalent seconds, k)."""
        from oracle import geometry, msve, tae
        tree, p = self.tree, self.preset
        t0 = time.perf_counter()
        res = self._all(("step", leaf, qi))
        t1 = time.perf_counter()
        N = tree.num_nodes
        mass = [sum(r[1][i] for r in res) for i in range(N)]
        Nq, Mclose = res[0][2], [sum(r[3][i] for r in res) for i in range(N)]
        s = []
        for i in range(N):
            a = msve.attention_feature(mass[i], Mclose[i], Nq[i], p["L"], p["Hq"])
            s.append(float(np.float32(msve.msve_score(self.params["theta"], float(tree.v[i]),
                                                       float(tree.u[i]), a))))
        tree.active = [leaf]
        parent = [int(x) for x in tree.parent]
        d = geometry.depths(parent)
        dist = geometry.delta(parent, tree.active)
        ps = geometry.path_star(parent, tree.active)
        st, k, _ = tae.allocate(self.params["alloc_mode"], s, d, dist, [i in ps for i in range(N)],
                                [False] * N, [int(x) for x in tree.span_len], self.params, budget)
        t2 = time.perf_counter()
        ev = self._all(("evict", leaf, k))
        t3 = time.perf_counter()
        serial = sum(r[0] for r in res) + (t2 - t1) + sum(r[0] for r in ev)
        return t3 - t0, serial, k

    def close(self):
        for c in self.conns:
            try:
                c.send(("quit",))
            except Exception:
                pass
        for pr in self.procs:
            pr.join(timeout=5)


def oracle_host_run(config, seed, warmup, steps, K, V, q_warm, q_step, warm_order, leaves,
                    budget, target_s=60.0, k_gpu=None):
    """Time the oracle fleet on the bench's workload: warm-up (untimed), then W + K steps
    (restore → step), the first W untimed; stops early (≥ 1 timed step) past target_s."""
    t_begin = time.perf_counter()
    fleet = OracleFleet(config, seed, K, V, q_warm, q_step)
    try:
        t_warm = fleet.warmup(warm_order)
        fleet.snapshot()
        times, serial, ks = [], [], []
        t_loop = time.perf_counter()
        for i in range(warmup + steps):
            dt, ser, k = fleet.step(leaves[i % 2], i % 2, budget)
            if i >= warmup:
                times.append(dt)
                serial.append(ser)
                ks.append(k)
            if time.perf_counter() - t_loop > target_s and times:
                break
    finally:
        fleet.close()
    T = fleet.tree.total_tokens
    t_step = statistics.median(times)
    same_k = None if k_gpu is None else all(k == k_gpu[j % 2] for j, k in enumerate(ks))
    return {"value": T / t_step, "ms_per_step": t_step * 1e3, "cores": fleet.cores,
            "steps_timed": len(times), "single_thread_equiv_tokens_per_s": T / statistics.median(serial),
            "cpu_model": _cpu_model(), "host_cores": _host_cores(),
            "wall_s": time.perf_counter() - t_begin, "warmup_s": t_warm, "k_equals_gpu": same_k,
            "sample": (f"{config}: the whole step on the whole workload ({fleet.tree.num_nodes} "
                       f"nodes, {T} tokens, all {fleet.preset['L'] * fleet.preset['H']} (layer, "
                       f"KV-head) rows): decode attention + score + node mass (rows: "
                       f"{fleet.cores} worker processes over layers) + MSVE + allocate (once) + "
                       f"evict; after the GPU arm's leaf-cycling warm-up ({len(warm_order)} steps, "
                       f"same queries); median of {len(times)} timed steps (wall clock incl. IPC)")}


def bench_inputs(config, seed, device):
    """The GPU arm's seeded inputs, on the host: K/V, the warm-up queries (leaf-cycling
    order, 4 steps per leaf) and the two step queries (workload.Scenario.queries)."""
    import torch
    import synth
    from paper_2605_22106_b200 import workload
    p = workload.PRESETS[config]
    tree = workload.build_tree(p, seed)
    K, V, E = synth.make_kv(p["L"], p["H"], tree.total_tokens, p["d"], p["dtype"], seed,
                            tree.span_start, tree.span_len, device=device)
    order = [leaf for leaf in workload.leaf_cycle_order(tree, seed) for _ in range(4)]

    def q(step):
        return synth.make_queries(1, p["L"], p["Hq"], p["d"], p["dtype"],
                                  workload.query_seed(seed, step), E, device=device).float().cpu()
    q_warm = [q(j) for j in range(len(order))]
    q_step = [q(10_000 + i) for i in range(2)]
    leaves = sorted(synth.leaves_of(tree), key=lambda x: -float(tree.v[x]))[:2]
    B = int(math.floor(p["rho"] * tree.total_tokens))
    return K.float().cpu(), V.float().cpu(), q_warm, q_step, order, leaves, B


# ---------------------------------------------------------------- GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--impl", default="arbor", choices=["arbor", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-steps", type=int, default=0,
                    help="just run N steps (for ncu launch lists); no JSON")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    from paper_2605_22106_b200 import workload
    from paper_2605_22106_b200.arbor import nccl_unique_id

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", init_method="env://", device_id=dev)
        pg = dist
    preset = workload.PRESETS[args.config]
    H = preset["H"]
    if H % ws:
        raise SystemExit(f"{H} KV heads do not split over {ws} GPUs")
    hc = H // ws
    nid = None
    if ws > 1:
        buf = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            buf.copy_(torch.frombuffer(bytearray(nccl_unique_id()), dtype=torch.uint8))
        pg.broadcast(buf, 0)
        nid = bytes(buf.cpu().numpy().tobytes())

    if args.config == "c3":
        return run_c3(args, dev, rank, ws, hc, nid, pg)
    sc = workload.setup(args.config, args.seed, kv_head_begin=rank * hc, kv_head_count=hc,
                        rank=rank, world_size=ws, nccl_id=nid, profile=True, device=dev)
    ctx, tree = sc.ctx, sc.tree
    workload.warmup_leaf_cycling(sc)
    import synth
    leaves = sorted(synth.leaves_of(tree), key=lambda x: -float(tree.v[x]))[:2]
    B = sc.budget
    N = tree.num_nodes
    nA = 1
    qs = [sc.queries(10_000 + i, nA) for i in range(2)]
    out = torch.empty_like(qs[0])
    lse = torch.empty((nA, ctx.L, ctx.Hq), dtype=torch.float32, device=dev)
    s_buf = torch.empty(N, dtype=torch.float32, device=dev)
    k_buf = torch.empty(N, dtype=torch.int32, device=dev)
    # full-retention snapshot (restored between steps, outside the timed region)
    snap_k, snap_v = ctx.k_pool.clone(), ctx.v_pool.clone()
    snap_pos, snap_A = ctx.pos_pool.clone(), ctx.score.clone()
    ctx.arbor_save_state(0)
    cached = int(np.asarray(tree.span_len).sum())
    trees = []
    from paper_2605_22106_b200.arbor import TreeArgs
    for leaf in leaves:
        tree.active = [leaf]
        trees.append(TreeArgs.from_tree(tree))
    stream = torch.cuda.current_stream(dev)

    # After the restore copies, a 256 MB read pass evicts their dirty lines from the 126 MB
    # L2 (write-backs happen there, untimed): each timed step starts from a flushed, clean
    # L2 instead of paying for the restore's write-backs (C2 a9 27.3 -> 23.3 us, A/B).
    read_flush = os.environ.get("ARBOR_BENCH_READ_FLUSH", "1") == "1"
    flush_buf = torch.ones(64 << 20, dtype=torch.float32, device=dev) if read_flush else None

    def restore():
        ctx.k_pool.copy_(snap_k)
        ctx.v_pool.copy_(snap_v)
        ctx.pos_pool.copy_(snap_pos)
        ctx.score.copy_(snap_A)
        ctx.arbor_load_state(0)
        if read_flush:      # evict the restore's dirty lines before the timed step
            flush_buf.sum()

    two_call = os.environ.get("ARBOR_BENCH_TWO_CALL") == "1"

    def step(i):
        ta = trees[i % 2]
        q = qs[i % 2]
        if two_call:      # diagnostics: the unfused a9 → a2/a3 calls (three launches)
            ctx.arbor_tree_decode_attn(ta, q, out, lse)
            ctx.arbor_score(ta, q, lse, s_buf)
        else:
            ctx.arbor_decode_step(ta, q, out, lse, s_buf)     # a9 + a2 + a3 (f2: two launches)
        ctx.arbor_allocate(ta, s_buf, B, k_buf)
        ctx.arbor_evict(ta, k_buf)

    if args.profile_steps:
        # for ncu: --nvtx --nvtx-include "bench_step/" selects exactly the step's kernels
        for i in range(args.profile_steps):
            restore()
            torch.cuda.synchronize()
            torch.cuda.nvtx.range_push("bench_step")
            step(i)
            torch.cuda.synchronize()
            torch.cuda.nvtx.range_pop()
        return

    for i in range(max(3, args.warmup)):
        restore()
        step(i)
    torch.cuda.synchronize()
    ctx.arbor_sync()

    # ---------------- timed region: K steps, each bracketed by CUDA events.  The library's
    # per-stage events are OFF here (a timing event costs the stream ~3 µs on B200); the
    # per-kernel durations come from a second, identical pass with them on (below).
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    stage_ms = {k: [] for k in ("attn", "attn_merge", "score_accum", "node_mass", "msve",
                                "allreduce", "geometry", "allocate", "evict_plan",
                                "select_compact", "compact_move")}
    launches = 0
    clocks = ClockSampler(local)
    ctx.arbor_set_profiling(False)
    if pg is not None:
        pg.barrier()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.2)
    for i in range(args.steps):            # no host sync inside: the host runs ahead
        restore()
        l0 = ctx.arbor_launch_count()
        ev[i][0].record(stream)
        step(i)
        ev[i][1].record(stream)
        launches += ctx.arbor_launch_count() - l0
    torch.cuda.synchronize()
    clk = clocks.stop()
    if pg is not None:
        pg.barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    # ---------------- per-kernel pass: the same K steps with the stage events on
    ctx.arbor_set_profiling(True)
    torch.cuda.synchronize()
    ctx.arbor_reset_stage_times()
    for i in range(args.steps):
        restore()
        step(i)
    torch.cuda.synchronize()
    st = ctx.arbor_stage_times()           # mean CUDA-event duration of each kernel stage
    for k in stage_ms:
        stage_ms[k] = [st[k]] * 2
    ctx.arbor_set_profiling(False)
    tot_ms = sum(step_ms)
    if pg is not None:
        t = torch.tensor([tot_ms], dtype=torch.float64, device=dev)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        tot_ms = float(t.item())
    ms_per_step = tot_ms / args.steps
    value = cached * args.steps / (tot_ms / 1e3)

    # ---------------- CUDA-Graph pass (SURVEY §8(d) timing protocol: eager AND graph-captured
    # steps): the step of each active leaf captured once (arbor_capture_begin/end), replayed
    # K times from the restored state; the restores stay eager, outside the timed region.
    graph_res = None
    if os.environ.get("ARBOR_BENCH_GRAPH", "1") == "1" and not two_call:
        graphs = []
        try:
            for i in range(2):
                restore()
                torch.cuda.synchronize()
                ctx.arbor_capture_begin()
                step(i)
                graphs.append(ctx.arbor_capture_end())
            # a replay must leave what the eager step leaves (k, s, the kept K/V)
            restore()
            step(0)
            torch.cuda.synchronize()
            k_e, s_e, kp_e = k_buf.clone(), s_buf.clone(), ctx.k_pool.view(torch.int16).sum(dtype=torch.int64)
            restore()
            ctx.arbor_graph_launch(graphs[0])
            torch.cuda.synchronize()
            same = bool(torch.equal(k_buf, k_e) and torch.equal(s_buf, s_e) and
                        int(ctx.k_pool.view(torch.int16).sum(dtype=torch.int64)) == int(kp_e))
            for i in range(max(3, args.warmup)):
                restore()
                ctx.arbor_graph_launch(graphs[i % 2])
            gev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(args.steps)]
            torch.cuda.synchronize()
            for i in range(args.steps):
                restore()
                gev[i][0].record(stream)
                ctx.arbor_graph_launch(graphs[i % 2])
                gev[i][1].record(stream)
            torch.cuda.synchronize()
            g_tot = sum(a.elapsed_time(b) for a, b in gev)
            if pg is not None:
                t = torch.tensor([g_tot], dtype=torch.float64, device=dev)
                pg.all_reduce(t, op=pg.ReduceOp.MAX)
                g_tot = float(t.item())
            graph_res = {"value": cached * args.steps / (g_tot / 1e3), "unit": "tokens/s",
                         "ms_per_step": g_tot / args.steps, "replay_matches_eager": same,
                         "note": "one CUDA graph per active leaf (arbor_capture_begin/end), "
                                 "replayed after the same eager restore; device-timed like value"}
        except Exception as e:  # noqa: BLE001
            graph_res = {"error": str(e)}
        finally:
            for g in graphs:
                ctx.arbor_graph_destroy(g)

    # ---------------- algorithmic bytes for the roofline, from the
    # device state after one step from full retention (per active leaf)
    def alg_bytes(i):
        restore()
        step(i)
        torch.cuda.synchronize()
        rb = ctx.D * (2 if preset["dtype"] == "bf16" else 4)
        L, Hh, P = ctx.L, ctx.H, ctx.P
        byts = {"select": 0, "compact_move": 0, "moved_rows": 0}
        for j in range(N):
            kc, n, pages = ctx.arbor_read_node(j)
            if kc == n:
                continue
            ko = ctx.arbor_read_node_offset(j)
            idx = torch.as_tensor(pages, device=dev, dtype=torch.long)
            pos = ctx.pos_pool[:, idx].permute(0, 2, 1, 3).reshape(L, Hh, -1)[:, :, ko:ko + kc]
            # from full retention the kept window is slots n − k_cur … n − 1 (Q23*): a row
            # moved iff its position is not its slot
            moved = int((pos.long() != torch.arange(n - kc, n, device=dev)).sum().item())
            # select, per (row, changed node): pos + A of the k_cur kept slots (2 + 4 B each);
            # move, per moved row: K and V read + write (4·rb) and its pos tag (2 + 2 B)
            byts["select"] += L * Hh * 6 * n
            byts["compact_move"] += moved * (4 * rb + 4)
            byts["moved_rows"] += moved
        vis = 0
        for x in synth_path(tree.parent, leaves[i % 2]):
            vis += int(tree.span_len[x])
        rows = L * Hh
        # a9: K + V of every visible token-row, plus Q read and O written
        byts["attn"] = rows * vis * 2 * rb + nA * ctx.Hq * L * 2 * rb
        # a3: A changes only at visible tokens, so only the visible closed nodes' partial
        # masses are recomputed (4 B per visible token-row); the rest are cached
        byts["node_mass"] = rows * vis * 4
        # a9 + a2 + a3 fused (a2 reuses a9's logits, so the K read is shared): a9's bytes +
        # the read-modify-write of A (8 B) + the node-mass read (4 B) per visible token-row
        byts["attn_score"] = byts["attn"] + rows * vis * 8 + byts["node_mass"]
        return byts

    ab = [alg_bytes(0), alg_bytes(1)]
    peak, peak_src = peaks()

    def kstat(name, bytes_fn):
        t_ms = []
        for i, x in enumerate(stage_ms[name]):
            t_ms.append(x)
        avg = statistics.mean(t_ms) if t_ms else float("nan")
        b = statistics.mean(bytes_fn(i) for i in range(2))
        gbs = b / (avg / 1e3) / 1e9 if avg > 0 else float("nan")
        return {"ms": avg, "bytes": b, "GBps": gbs, "frac_measured": gbs / peak,
                "frac_nominal": gbs / NOMINAL_HBM}

    if stage_ms["compact_move"][0] > 0:       # split select → move kernels
        kernels = {"compact_move": kstat("compact_move", lambda i: ab[i]["compact_move"]),
                   "select": kstat("select_compact", lambda i: ab[i]["select"])}
        top_name, top_desc = "compact_move", "compact_move (a6)"
    else:                                     # one select+compact kernel (default)
        kernels = {"select_compact": kstat("select_compact",
                                           lambda i: ab[i]["select"] + ab[i]["compact_move"])}
        top_name, top_desc = "select_compact", "select_move_ws (a5+a6, warp-specialised)"
    kernels["attn_partial"] = kstat("attn", lambda i: ab[i]["attn"])
    if stage_ms["node_mass"][0] > 0:          # unfused a3 (multi-rank runs)
        kernels["node_mass"] = kstat("node_mass", lambda i: ab[i]["node_mass"])
    # a9 + a2 + a3 as one unit (arbor_decode_step: attention kernel + merge/score kernel)
    t_as = sum(statistics.mean(stage_ms[k]) for k in ("attn", "attn_merge", "score_accum",
                                                       "node_mass", "msve"))
    b_as = statistics.mean(ab[i]["attn_score"] for i in range(2))
    kernels["attn_score_fused"] = {"ms": t_as, "bytes": b_as, "GBps": b_as / (t_as / 1e3) / 1e9,
                                   "frac_measured": b_as / (t_as / 1e3) / 1e9 / peak,
                                   "frac_nominal": b_as / (t_as / 1e3) / 1e9 / NOMINAL_HBM,
                                   "stages": ["attn", "attn_merge", "score_accum", "node_mass", "msve"]}
    top = kernels[top_name]
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        try:
            pj = json.load(open(prof))
            ent = pj.get(args.config, {}).get(top_name)
            if ent:
                traffic = ent["dram_bytes_per_launch"]
        except Exception:
            traffic = None
    roofline = {"kernel": top_desc, "bound": "hbm", "achieved": top["GBps"],
                "peak": peak, "unit": "GB/s", "frac": top["GBps"] / peak,
                "frac_of_nominal_8TBps": top["GBps"] / NOMINAL_HBM, "traffic": traffic,
                "peak_source": peak_src, "alg_bytes_per_launch": top["bytes"],
                "ms_per_launch": top["ms"]}

    # ---------------- e2e: host buffers through the public API (pinned H2D q, D2H k, s)
    q_host = [q.cpu().pin_memory() for q in qs]
    # s and k side by side in one device buffer, read back with one copy that runs on a
    # second stream while the eviction (which needs neither) runs: both are final after
    # arbor_allocate (ARBOR_BENCH_E2E_OVERLAP=0: two copies after the eviction)
    sk_dev = torch.empty(2 * N, dtype=torch.int32, device=dev)
    s_e, k_e = sk_dev[:N].view(torch.float32), sk_dev[N:]
    sk_host = torch.empty(2 * N, dtype=torch.int32).pin_memory()
    overlap = os.environ.get("ARBOR_BENCH_E2E_OVERLAP", "1") == "1"
    cs = torch.cuda.Stream(dev)
    q_dev = torch.empty_like(qs[0])
    e2e_ms = []
    for i in range(args.steps):
        restore()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        q_dev.copy_(q_host[i % 2], non_blocking=True)
        ta = trees[i % 2]
        ctx.arbor_decode_step(ta, q_dev, out, lse, s_e)
        ctx.arbor_allocate(ta, s_e, B, k_e)
        if overlap:
            cs.wait_stream(stream)
            with torch.cuda.stream(cs):
                sk_host.copy_(sk_dev, non_blocking=True)
            ctx.arbor_evict(ta, k_e)
            stream.wait_stream(cs)
        else:
            ctx.arbor_evict(ta, k_e)
            sk_host[N:].copy_(k_e, non_blocking=True)
            sk_host[:N].copy_(sk_dev[:N], non_blocking=True)
        b.record(stream)
        b.synchronize()
        e2e_ms.append(a.elapsed_time(b))
    e2e_tot = sum(e2e_ms)
    if pg is not None:
        t = torch.tensor([e2e_tot], dtype=torch.float64, device=dev)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        e2e_tot = float(t.item())
    e2e = {"value": cached * args.steps / (e2e_tot / 1e3), "unit": "tokens/s",
           "h2d_bytes_per_step": int(qs[0].numel() * qs[0].element_size()),
           "d2h_bytes_per_step": int(N * 8)}

    # ---------------- rehydration (a7/a8): backtrack into the evicted subtree
    rehyd = None
    try:
        restore()
        step(0)
        other = [x for x in synth.leaves_of(tree) if x not in leaves]
        tree.active = [other[len(other) // 2]]
        ta = TreeArgs.from_tree(tree)
        path = synth_path(tree.parent, tree.active[0])
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        r0 = ctx.arbor_read_counters()[0]
        # PCIe bytes: the evicted rows (n − k_cur) of the path nodes (Q23r: the
        # kept rows are restored within HBM)
        miss = sum(int(tree.span_len[x]) - ctx.arbor_read_node(x)[0] for x in path)
        nbytes = miss * ctx.L * ctx.H * ctx.D * 2 * (2 if preset["dtype"] == "bf16" else 4)
        torch.cuda.synchronize()
        a.record(stream)
        ctx.arbor_rehydrate(ta, path)
        b.record(ctx.side)                      # the copy runs on the side stream
        b.synchronize()
        r1 = ctx.arbor_read_counters()[0]
        ms = a.elapsed_time(b)
        rehyd = {"nodes_rehydrated": int(r1 - r0), "ms": ms, "bytes": nbytes,
                 "PCIe_GBps": nbytes / (ms / 1e3) / 1e9 if ms > 0 else None,
                 "note": "zero-copy reads of the pinned-host stash by a side-stream kernel; "
                         "bytes = full spans of the path nodes with k_cur < n"}
    except Exception as e:  # pragma: no cover
        rehyd = {"error": str(e)}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        # the oracle on the host cores, same inputs / warm-up / step as this arm (sc.K, sc.V
        # are this process's device tensors; queries regenerated with the same seeds)
        Kh, Vh = sc.K.float().cpu(), sc.V.float().cpu()
        _, _, q_warm, q_step, order, leaves_h, B_h = bench_inputs(args.config, args.seed, dev)
        k_gpu = []
        for i in range(2):
            restore()
            step(i)
            torch.cuda.synchronize()
            k_gpu.append(k_buf.cpu().tolist())
        r = oracle_host_run(args.config, args.seed, 1, 3, Kh, Vh, q_warm, q_step, order,
                            leaves_h, B_h, target_s=30.0, k_gpu=k_gpu)
        del Kh, Vh
        cpu = {"value": r["value"], "unit": "tokens/s", "cores": r["cores"], "kind": "oracle",
               "sample": r["sample"], "cpu_model": r["cpu_model"], "host_cores": r["host_cores"],
               "single_thread_equiv_tokens_per_s": r["single_thread_equiv_tokens_per_s"],
               "k_equals_gpu": r["k_equals_gpu"], "wall_s": r["wall_s"]}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": ws,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": preset["dtype"], "data": "synthetic",
                "config": dict(workload_config(args.config, ws), cached_tokens=cached, budget=B,
                               nodes=N, step="a9 attn + a2 score + a3 mass/MSVE + a1 geometry + "
                                            "a4 allocate + a5/a6 select+compact (+a10 all-reduce)"),
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "graph": graph_res,
                "gpu_launches": launches, "gpu_launches_per_step": launches / args.steps,
                "clocks": clk, "kernels": kernels, "kernel_timing": "second pass of the same K steps with per-stage CUDA events on the launching stream (each event pair adds ~3 us of stream time; included, so per-kernel GB/s are conservative)",
                "stage_ms_median": {k: statistics.median(v) for k, v in stage_ms.items() if v},
                "step_ms_p10_p50_p90": [float(np.percentile(step_ms, q)) for q in (10, 50, 90)],
                "rehydrate": rehyd,
                "decode_attn": {"GBps": kernels["attn_partial"]["GBps"],
                                "frac_measured": kernels["attn_partial"]["frac_measured"],
                                "frac_nominal": kernels["attn_partial"]["frac_nominal"]}}
        print(json.dumps(line), flush=True)
    if pg is not None:
        pg.barrier()
        pg.destroy_process_group()


def c3_traffic():
    """DRAM bytes per launch of the C3 attention kernel from the committed ncu capture
    (profiles/ncu_traffic.json, c3/attn), or None."""
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))["c3"]["attn"]["dram_bytes_per_launch"]
    except Exception:
        return None


def run_c3(args, dev, rank, ws, hc, nid, pg):
    """configs[2]: the DPTS frontier.  16 active leaves under distinct
    level-2 parents of the 8B-shaped depth-4 × width-5 tree, ρ = 0.5 (B = 9,984 fixed while
    the tree grows).  One step = one transition (4 of the 16 leaves replaced: backtracks into
    possibly evicted subtrees; a fresh open child under each new leaf) = Alg. 2's order:
    rehydrate the new Path* (a8, side stream) → allocate (a1+a4) → evict (a5+a6), the last two
    overlapping the copy, followed by 8 decode steps (append one token to every open child;
    a9 over the shared tree; a2+a3).  `value` = cached tokens at the transition ÷ the
    allocate + evict device time; rehydration (PCIe) is reported separately, with how long
    the first decode waits for it; decode attention is reported with tree sharing (a shared
    node is read once for all leaves below it)."""
    import torch
    import synth
    from paper_2605_22106_b200 import workload
    from paper_2605_22106_b200.arbor import TreeArgs
    # the context is sized for the whole run: pages and positions for every open child, and
    # per node only one child's growth (workload.dpts_sizing)
    K, W, D = args.steps, max(3, args.warmup), 8
    transitions = K + W
    extra_nodes, extra_tokens, node_extra = workload.dpts_sizing(transitions, D)
    sc = workload.setup("c3", args.seed, kv_head_begin=rank * hc, kv_head_count=hc, rank=rank,
                        world_size=ws, nccl_id=nid, profile=True, device=dev,
                        extra_tokens=extra_tokens, extra_nodes=extra_nodes, max_active=16,
                        node_extra_tokens=node_extra)
    ctx, tree = sc.ctx, sc.tree
    workload.warmup_leaf_cycling(sc)
    run = workload.DptsRun(sc, n_active=16, transitions=transitions, swap=4, decode_steps=D,
                           seed=args.seed)
    stream = torch.cuda.current_stream(dev)
    preset = sc.preset
    rb = ctx.D * (2 if preset["dtype"] == "bf16" else 4)
    rows = ctx.L * ctx.H
    ctx.arbor_set_profiling(False)
    rec = []
    clocks = ClockSampler(dev.index if dev.index is not None else 0)
    serial_rehyd = os.environ.get("ARBOR_BENCH_C3_SERIAL") == "1"
    # ~300 µs of device sleep before each transition (ARBOR_BENCH_RUN_AHEAD=0: none)
    run_ahead_cycles = int(float(os.environ.get("ARBOR_BENCH_RUN_AHEAD", "1")) * 300e-6 *
                           torch.cuda.get_device_properties(dev).clock_rate * 1e3) \
        if hasattr(torch.cuda.get_device_properties(dev), "clock_rate") else 600000
    schedule = [run.base_leaves] + run.schedule
    if pg is not None:
        pg.barrier()
    torch.cuda.synchronize()
    clocks.start()
    for t, leaves in enumerate(schedule[:transitions]):
        timed = t >= W
        run.activate(leaves)
        ta = TreeArgs.from_tree(tree)
        cached = sum(ctx.arbor_read_node(x)[0] for x in range(tree.num_nodes))
        r0 = ctx.arbor_read_counters()[0]
        k = run.k_buf[:tree.num_nodes]
        path = [x for x in run.path_union() if not tree.is_open[x]]
        rbytes = 0                                  # PCIe bytes: the evicted rows only (Q23r)
        for x in path:
            kc_x, n_x, _ = ctx.arbor_read_node(x)
            rbytes += (n_x - kc_x) * rows * 2 * rb
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        rs, rd = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        l0 = ctx.arbor_launch_count()
        # Alg. 2 Transition: rehydrate Path* (side stream), then allocate + evict on the main
        # stream while the copy runs; the first decode waits for the copy
        # host run-ahead (odd transitions): a device sleep queued first lets the host enqueue
        # the whole transition (~50 µs of API calls) before the device reaches it, as the C2
        # loop does by never synchronising — their events time the device, not the host's
        # enqueue; the even transitions run without it and give `e2e` (host wall clock)
        gated = bool(run_ahead_cycles) and t % 2 == 1
        if gated:
            torch.cuda._sleep(run_ahead_cycles)
        w0 = time.perf_counter()
        rs.record(stream)
        ctx.arbor_rehydrate(ta, path)
        rd.record(ctx.side)                         # the copy's completion (side stream)
        if serial_rehyd:                            # diagnostics: no overlap with the copy
            stream.wait_event(rd)
        e[0].record(stream)
        ctx.arbor_allocate(ta, None, run.budget, k)
        e[1].record(stream)
        ctx.arbor_evict(ta, k)
        e[2].record(stream)
        e[2].synchronize()
        wall = time.perf_counter() - w0
        e[3].record(stream)                         # where the first decode would start
        torch.cuda.synchronize()
        rwall = time.perf_counter() - w0
        launches = ctx.arbor_launch_count() - l0
        r1 = ctx.arbor_read_counters()[0]
        # a9 bytes with tree sharing: K+V of every kept slot of the union of the active paths
        vis = sum(ctx.arbor_read_node(x)[0] for x in run.path_union())
        attn_bytes = rows * vis * 2 * rb + len(tree.active) * ctx.Hq * ctx.L * 2 * rb
        dec = []
        for _ in range(D):
            for ch in tree.active:
                run._append(ch)
            q = sc.queries(1_000_000 + run.step, len(tree.active))
            run.step += 1
            out = torch.empty_like(q)
            lse = torch.empty((len(tree.active), ctx.L, ctx.Hq), dtype=torch.float32, device=dev)
            tq = TreeArgs.from_tree(tree)
            d = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            d[0].record(stream)
            ctx.arbor_decode_step(tq, q, out, lse)
            d[1].record(stream)
            d[2].record(stream)
            dec.append(d)
        torch.cuda.synchronize()
        if timed:
            rec.append(dict(gated=gated, cached=cached, alloc=e[0].elapsed_time(e[1]),
                            evict=e[1].elapsed_time(e[2]), rehyd=rs.elapsed_time(rd),
                            rehyd_wait=max(0.0, e[2].elapsed_time(rd)),
                            trans=e[0].elapsed_time(e[2]), wall=wall, nrehyd=r1 - r0,
                            rehyd_bytes=rbytes, launches=launches, attn=[x[0].elapsed_time(x[1]) for x in dec],
                            score=[x[1].elapsed_time(x[2]) for x in dec], attn_bytes=attn_bytes))
    clk = clocks.stop()
    rec_e2e = [r for r in rec if not r["gated"]] or rec
    rec = [r for r in rec if r["gated"]] or rec     # device-timed transitions
    # per-kernel pass: one more transition + its decode steps with the library's stage
    # events on (kernel-only durations), and the host time of each API call
    ctx.arbor_set_profiling(True)
    ctx.arbor_reset_stage_times()
    host_ms = {"allocate": [], "evict": [], "attn": [], "score": []}
    for leaves in schedule[transitions:transitions + 1] or schedule[-1:]:
        run.activate(leaves)
        ta = TreeArgs.from_tree(tree)
        k = run.k_buf[:tree.num_nodes]
        torch.cuda.synchronize()
        ctx.arbor_rehydrate(ta, [x for x in run.path_union() if not tree.is_open[x]])
        h = time.perf_counter(); ctx.arbor_allocate(ta, None, run.budget, k)
        host_ms["allocate"].append((time.perf_counter() - h) * 1e3)
        h = time.perf_counter(); ctx.arbor_evict(ta, k)
        host_ms["evict"].append((time.perf_counter() - h) * 1e3)
        for _ in range(D):
            for ch in tree.active:
                run._append(ch)
            q = sc.queries(2_000_000 + run.step, len(tree.active))
            run.step += 1
            out = torch.empty_like(q)
            lse = torch.empty((len(tree.active), ctx.L, ctx.Hq), dtype=torch.float32, device=dev)
            tq = TreeArgs.from_tree(tree)
            torch.cuda.synchronize()
            h = time.perf_counter(); ctx.arbor_decode_step(tq, q, out, lse)
            host_ms["attn"].append((time.perf_counter() - h) * 1e3)
            host_ms["score"].append(0.0)
        torch.cuda.synchronize()
    stage = ctx.arbor_stage_times()
    ctx.arbor_set_profiling(False)
    tot_ms = sum(r["alloc"] + r["evict"] for r in rec)
    if pg is not None:
        tt = torch.tensor([tot_ms], dtype=torch.float64, device=dev)
        pg.all_reduce(tt, op=pg.ReduceOp.MAX)
        tot_ms = float(tt.item())
    cached_tot = sum(r["cached"] for r in rec)
    value = cached_tot / (tot_ms / 1e3)
    peak, peak_src = peaks()
    attn_ms = statistics.median([x for r in rec for x in r["attn"]])   # whole decode step
    attn_b = statistics.mean(r["attn_bytes"] for r in rec)
    attn_gbs = attn_b / (attn_ms / 1e3) / 1e9
    # the attention kernel alone: its mean launch duration from the per-stage pass
    kern_ms = stage.get("attn") or attn_ms
    kern_gbs = attn_b / (kern_ms / 1e3) / 1e9
    wall_tot = sum(r["wall"] for r in rec_e2e)
    nodes_n = tree.num_nodes
    line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": ws, "steps": K,
            "warmup": W, "ms_per_step": tot_ms / len(rec), "timed_transitions": len(rec),
            "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": preset["dtype"], "data": "synthetic",
            "config": dict(workload_config("c3", ws), budget=run.budget, active_leaves=16,
                           decode_steps_per_transition=D,
                           step="one DPTS transition (Alg. 2 order): a8 rehydrate issued on the "
                                "side stream -> a1+a4 allocate -> a5+a6 evict (timed); then 8 decode steps of arbor_decode_step "
                                "(a9 + a2/a3, reported separately)"),
            "roofline": {"kernel": "attn_tc (a9, 16 leaves, tree-shared tiles)", "bound": "hbm",
                         "achieved": kern_gbs, "peak": peak, "unit": "GB/s",
                         "frac": kern_gbs / peak, "frac_of_nominal_8TBps": kern_gbs / NOMINAL_HBM,
                         "traffic": c3_traffic(), "peak_source": peak_src,
                         "alg_bytes_per_launch": attn_b, "ms_per_launch": kern_ms,
                         "decode_step_GBps": attn_gbs, "decode_step_ms": attn_ms,
                         "note": "achieved / ms_per_launch: the attention kernel's mean launch "
                                 "duration (per-stage CUDA events, incl. ~3 us event cost); "
                                 "decode_step_*: arbor_decode_step = attention + merge/score "
                                 "kernel; bytes: K/V (shared nodes once) + Q/O"},
            "cpu_baseline": None,
            "e2e": {"value": sum(r["cached"] for r in rec_e2e) / wall_tot, "unit": "tokens/s",
                    "h2d_bytes_per_step": int(nodes_n * 25 + 64), "d2h_bytes_per_step": 16,
                    "note": "host wall clock of the transition calls incl. tree upload and sync "
                            "(the transitions without host run-ahead)",
                    "wall_us_p50": statistics.median(r["wall"] * 1e6 for r in rec_e2e),
                    "device_us_p50": statistics.median(r["trans"] * 1e3 for r in rec_e2e)},
            "timing_note": "value and the per-transition device times come from the transitions "
                           "queued behind a ~300 us device sleep (host run-ahead, as in the C2 "
                           "loop); e2e from the others (ARBOR_BENCH_RUN_AHEAD=0: no sleep)",
            "gpu_launches": sum(r["launches"] for r in rec),
            "gpu_launches_per_step": statistics.mean(r["launches"] for r in rec), "clocks": clk,
            "transition_us_p10_p50_p90": [float(np.percentile([r["trans"] * 1e3 for r in rec], q))
                                          for q in (10, 50, 90)],
            "allocate_us_p50": statistics.median(r["alloc"] * 1e3 for r in rec),
            "evict_us_p50": statistics.median(r["evict"] * 1e3 for r in rec),
            "rehydrate": {"ms_p50": statistics.median(r["rehyd"] for r in rec),
                          "bytes_per_transition": statistics.mean(r["rehyd_bytes"] for r in rec),
                          "PCIe_GBps": (sum(r["rehyd_bytes"] for r in rec) /
                                        (sum(r["rehyd"] for r in rec) / 1e3) / 1e9)
                                       if sum(r["rehyd"] for r in rec) > 0 else None,
                          "decode_wait_ms_p50": statistics.median(r["rehyd_wait"] for r in rec),
                          "ready_before_next_decode": sum(1 for r in rec if r["rehyd_wait"] == 0.0),
                          "transitions": len(rec),
                          "note": "side-stream zero-copy reads of the pinned-host stash, issued before allocate + evict (Alg. 2 order) and overlapping them; ms_p50 = CUDA events (rehydrate call on the main stream -> copy done on the side stream); decode_wait = how long the first decode after the transition waits for the copy"},
            "rehydrations_per_transition": statistics.mean(r["nrehyd"] for r in rec),
            "decode_attn_us_p50": attn_ms * 1e3,
            "decode_attn_GBps": attn_gbs,
            "score_us_p50": statistics.median(x for r in rec for x in r["score"]) * 1e3,
            "stage_ms_mean": {k: v for k, v in stage.items() if v},
            "host_api_ms_median": {k: statistics.median(v) for k, v in host_ms.items() if v},
            "decode_tokens_per_s": 16 / ((attn_ms + statistics.median(
                x for r in rec for x in r["score"])) / 1e3)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if pg is not None:
        pg.barrier()
        pg.destroy_process_group()


def synth_path(parent, leaf):
    out = []
    x = int(leaf)
    while x >= 0:
        out.append(x)
        x = int(parent[x])
    return out[::-1]


if __name__ == "__main__":
    main()
