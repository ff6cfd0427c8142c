"""Synthetic ToT / DPTS workloads driven through libarbor (BASELINE.json configs).

Presets C1–C5 concretise BASELINE.json ``configs`` (the paper's Config-S/L shapes,
PAPER.md §5.1, on Llama-3.1-8B / Qwen2.5-32B-shaped KV).  Inputs are seeded and
synthetic (``synth``); every step runs in the library's kernels.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

import synth
from .arbor import ArborKV, make_params

PRESETS = {
    # configs[0]: tiny tree, depth 3 branching 2, 32 tokens/node, 1 layer, 2 KV heads, d 64, fp32
    "c1": dict(tree=("full", 3, 2, 32), L=1, H=2, Hq=2, d=64, dtype="f32", P=8, rho=0.5,
               params=dict(k_min=2, l_tail=2, r_min=0.0, eta=1.0), active="node3"),
    # configs[1]: Llama-3.1-8B-shaped KV, ToT depth 4 width 5, 25% budget
    "c2": dict(tree=("full", 4, 5, 128), L=32, H=8, Hq=32, d=128, dtype="bf16", P=16, rho=0.25,
               params={}, active="highest_v"),
    # configs[2]: DPTS frontier, 16 active branches on 8B-shaped KV, 50% budget
    "c3": dict(tree=("full", 4, 5, 128), L=32, H=8, Hq=32, d=128, dtype="bf16", P=16, rho=0.5,
               params={}, active="dpts16"),
    # configs[3]: Qwen2.5-32B-shaped GQA KV, deep tree (depth 8, width 4), 25% budget
    "c4": dict(tree=("search", 256, 4, 8, 128), L=64, H=8, Hq=40, d=128, dtype="bf16", P=16,
               rho=0.25, params={}, active="highest_v"),
    # configs[4]: budget sweep on 8B-shaped trees up to 64k tokens
    "c5": dict(tree=("search", 512, 3, 8, 128), L=32, H=8, Hq=32, d=128, dtype="bf16", P=16,
               rho=0.25, params={}, active="highest_v"),
}


def build_tree(preset: dict, seed: int = 0):
    kind = preset["tree"]
    if kind[0] == "full":
        t = synth.full_tree(kind[1], kind[2], kind[3], seed)
    else:
        t = synth.search_tree(kind[1], kind[2], kind[3], kind[4], seed)
    act = preset["active"]
    if act == "node3":
        t.active = [3]
    elif act == "highest_v":
        t.active = [synth.highest_v_leaf(t)]
    elif act == "dpts16":
        t.active = synth.dpts_initial_leaves(t, 16, seed)
    return t


def preset_params(preset: dict, **over):
    d = dict(preset["params"])
    d.update(over)
    return make_params(**d)


def make_context(preset: dict, tree, *, extra_tokens=0, extra_nodes=0, max_active=16,
                 params=None, layer_begin=0, layer_count=None, kv_head_begin=0,
                 kv_head_count=None, rank=0, world_size=1, nccl_id=None, profile=False,
                 page_margin=64, node_extra_tokens=None, external_reduce=False,
                 collective=False) -> ArborKV:
    """extra_tokens / extra_nodes: growth of the whole tree beyond the snapshot (pages, the
    position stream); node_extra_tokens: the most tokens any ONE node may grow to beyond
    the snapshot's largest node (int16 position tags per node; default extra_tokens)."""
    P = preset["P"]
    per_node = extra_tokens if node_extra_tokens is None else node_extra_tokens
    n = np.asarray(tree.span_len, np.int64)
    max_node = int(max(n.max(), 1))
    pages = int(sum(-(-int(x) // P) for x in n)) + -(-extra_tokens // P) + extra_nodes + page_margin
    max_tokens = int(tree.end_position() + extra_tokens + 8)
    return ArborKV(num_layers=preset["L"], num_kv_heads=preset["H"], num_q_heads=preset["Hq"],
                   head_dim=preset["d"], dtype=preset["dtype"], page_size=P, num_pages=pages,
                   max_nodes=tree.num_nodes + extra_nodes + 1,
                   max_node_tokens=max(max_node, 1) + max(per_node, 0) + 1,
                   max_active=max_active, max_tokens=max_tokens,
                   params=params if params is not None else preset_params(preset),
                   layer_begin=layer_begin, layer_count=layer_count, kv_head_begin=kv_head_begin,
                   kv_head_count=kv_head_count, rank=rank, world_size=world_size, nccl_id=nccl_id,
                   profile=profile, external_reduce=external_reduce, collective=collective)


def load_tree(ctx: ArborKV, tree, K, V):
    """Open, fill and close every node of a snapshot (prefill of the tree's KV).
    K, V: device [L][H][T][d] by absolute position (this rank's shard)."""
    for i in range(tree.num_nodes):
        a, n = int(tree.span_start[i]), int(tree.span_len[i])
        ctx.arbor_open_node(i, a)
        if n > 0:
            ctx.arbor_append_kv(i, K[:, :, a:a + n].contiguous(), V[:, :, a:a + n].contiguous())
        if not tree.is_open[i]:
            ctx.arbor_close_node(i)


def decode_step(ctx: ArborKV, tree, q, out=None, lse=None, fused=False):
    """One decode step for the active leaves: tree decode attention (a9) then score (a2/a3) —
    two calls, or (fused) the f2 call arbor_decode_step."""
    import torch
    nA = len(tree.active)
    if out is None:
        out = torch.empty_like(q)
    if lse is None:
        lse = torch.empty((nA, ctx.L, ctx.Hq), dtype=torch.float32, device=q.device)
    if fused:
        ctx.arbor_decode_step(tree, q, out, lse)
        return out, lse
    ctx.arbor_tree_decode_attn(tree, q, out, lse)
    ctx.arbor_score(tree, q, lse)
    return out, lse


def leaf_cycle_order(tree, seed: int):
    leaves = synth.leaves_of(tree)
    rng = np.random.default_rng(seed + 31337)
    return [int(x) for x in rng.permutation(leaves)]


def query_seed(seed: int, step: int) -> int:
    return seed * 1000003 + step


@dataclass
class Scenario:
    preset: dict
    tree: object
    ctx: ArborKV
    K: object          # this rank's shard [L][H_local][T][d]
    V: object
    E_full: object     # [L][H][d] directions of ALL heads (queries are drawn for all heads
    seed: int          # and sliced, so every world size sees identical inputs)
    kv_head_begin: int = 0
    steps: int = 0

    @property
    def budget(self) -> int:
        return int(math.floor(self.preset["rho"] * self.tree.total_tokens))

    def queries(self, step: int, n_active: int):
        p = self.preset
        q = synth.make_queries(n_active, p["L"], p["Hq"], p["d"], p["dtype"],
                               query_seed(self.seed, step), self.E_full, device=self.ctx.device)
        G = self.ctx.G
        h0 = self.kv_head_begin
        return q[:, :, h0 * G:(h0 + self.ctx.H) * G].contiguous()


def setup(preset_name: str, seed: int = 0, *, kv_head_begin=0, kv_head_count=None, rank=0,
          world_size=1, nccl_id=None, profile=False, extra_tokens=0, extra_nodes=0,
          params=None, max_active=16, device="cuda", node_extra_tokens=None,
          external_reduce=False, collective=False) -> Scenario:
    """Build the preset's tree, its seeded K/V (on the device), a context, and prefill it."""
    preset = PRESETS[preset_name]
    tree = build_tree(preset, seed)
    H = preset["H"]
    hc = kv_head_count if kv_head_count is not None else H
    K, V, E = synth.make_kv(preset["L"], H, tree.total_tokens, preset["d"], preset["dtype"], seed,
                            tree.span_start, tree.span_len, device=device)
    if hc != H:
        K = K[:, kv_head_begin:kv_head_begin + hc].contiguous()
        V = V[:, kv_head_begin:kv_head_begin + hc].contiguous()
    ctx = make_context(preset, tree, extra_tokens=extra_tokens, extra_nodes=extra_nodes,
                       max_active=max_active, params=params, kv_head_begin=kv_head_begin,
                       kv_head_count=hc, rank=rank, world_size=world_size, nccl_id=nccl_id,
                       profile=profile, node_extra_tokens=node_extra_tokens,
                       external_reduce=external_reduce, collective=collective)
    load_tree(ctx, tree, K, V)
    return Scenario(preset, tree, ctx, K, V, E, seed, kv_head_begin)


def warmup_leaf_cycling(sc: Scenario, steps_per_leaf: int = 4):
    """§8(c).1 item 10: every leaf is the sole active leaf for ``steps_per_leaf`` decode
    steps, in a seeded order, so every node accumulates mass from its own subtree."""
    saved = list(sc.tree.active)
    for leaf in leaf_cycle_order(sc.tree, sc.seed):
        sc.tree.active = [leaf]
        for _ in range(steps_per_leaf):
            q = sc.queries(sc.steps, 1)
            decode_step(sc.ctx, sc.tree, q)
            sc.steps += 1
    sc.tree.active = saved


# ---------------------------------------------------------------- C3: DPTS transition loop
def dpts_sizing(transitions: int, decode_steps: int = 8, n_active: int = 16, swap: int = 4):
    """Context growth of a DptsRun: (extra_nodes, extra_tokens, node_extra_tokens).  Every
    open child reserves child_cap = decode_steps·(transitions + 1) + 2 positions."""
    child_cap = decode_steps * (transitions + 1) + 2
    extra_nodes = n_active + swap * transitions + 4
    return extra_nodes, extra_nodes * child_cap + 64, child_cap



class DptsRun:
    """configs[2]: n_active leaves under distinct level-2
    parents; each transition replaces `swap` of them (backtracks into possibly evicted
    subtrees), opens a fresh child under every newly activated leaf (where decoding writes)
    and closes the children of deactivated leaves (Boundary); then
      rehydrate the new Path* (a7/a8, side stream) → allocate (a1+a4, with the last scores) →
    evict (a5+a6), followed by `decode_steps` decode steps (append one token to every open child; a9; a2/a3).
    The budget B = ⌊ρ·T_tot(base tree)⌋ stays fixed while the tree grows."""

    def __init__(self, sc: "Scenario", n_active=16, transitions=32, swap=4, decode_steps=8,
                 seed=0, on_append=None):
        import torch
        self.sc = sc
        self.torch = torch
        self.tree = sc.tree
        self.base_leaves = synth.dpts_initial_leaves(sc.tree, n_active, seed)
        self.schedule = synth.dpts_schedule(sc.tree, self.base_leaves, transitions, swap, seed)
        self.decode_steps = decode_steps
        self.budget = sc.budget
        self.child_of = {}            # active base leaf -> its open child node
        self.step = 0
        self.on_append = on_append
        self.log = []                 # ("append", node, pos) / ("close", node) / ("open", node, a)
        # every open child gets a reserved, disjoint range of the position stream
        self.child_cap = decode_steps * (transitions + 1) + 2
        self.next_pos = sc.tree.end_position()
        self.k_buf = torch.empty(sc.ctx.max_nodes, dtype=torch.int32, device=sc.ctx.device)

    def _kv_token(self, node: int, t: int):
        """Seeded K/V of one appended token of an open child: [L][H_local][1][d] (CPU-drawn
        for all heads, sliced to this rank's heads, so every world size sees the same data)."""
        p = self.sc.preset
        g = self.torch.Generator().manual_seed(int(self.sc.seed * 7_000_003 + node * 10_007 + t))
        shape = (p["L"], p["H"], 1, p["d"])
        k = self.torch.randn(shape, generator=g)
        v = self.torch.randn(shape, generator=g)
        h0, hc = self.sc.kv_head_begin, self.sc.ctx.H
        td = self.sc.ctx.tdtype
        return k[:, h0:h0 + hc].to(td).contiguous(), v[:, h0:h0 + hc].to(td).contiguous()

    def _append(self, node: int):
        ctx, tree = self.sc.ctx, self.tree
        t = int(tree.span_len[node])
        k, v = self._kv_token(node, t)
        ctx.arbor_append_kv(node, k.to(ctx.device), v.to(ctx.device))
        if self.on_append:
            self.on_append(node, int(tree.span_start[node]) + t, k, v)
        self.log.append(("append", node, int(tree.span_start[node]) + t))
        tree.span_len[node] += 1

    def activate(self, leaves):
        """Open children for newly active leaves, close those of deactivated leaves."""
        ctx, tree = self.sc.ctx, self.tree
        new = set(leaves)
        for leaf, ch in list(self.child_of.items()):
            if leaf not in new:
                if int(tree.span_len[ch]) == 0:    # never decoded: give it one token first
                    self._append(ch)
                ctx.arbor_close_node(ch)
                self.log.append(("close", ch))
                tree.is_open[ch] = 0
                del self.child_of[leaf]
        for leaf in leaves:
            if leaf not in self.child_of:
                a = self.next_pos
                self.next_pos += self.child_cap
                node = tree.add_node(leaf, a, 0, True, float(tree.v[leaf]), float(tree.u[leaf]))
                ctx.arbor_open_node(node, a)
                self.log.append(("open", node, a))
                self.child_of[leaf] = node
        tree.active = [self.child_of[l] for l in leaves]

    def path_union(self):
        tree = self.tree
        out = set()
        for leaf in tree.active:
            x = int(leaf)
            while x >= 0:
                out.add(x)
                x = int(tree.parent[x])
        return sorted(out)

    def transition(self, leaves):
        """Alg. 2 Transition: activate → rehydrate the new Path* (side stream,
        l.8-14) → allocate (last scores; 0.5 for never-scored nodes) → evict where k drops
        (l.15-21).  The allocation and eviction overlap the rehydration copy; the next decode
        waits for it."""
        ctx, tree = self.sc.ctx, self.tree
        self.activate(leaves)
        ctx.arbor_rehydrate(tree, [x for x in self.path_union() if not tree.is_open[x]])
        k = self.k_buf[:tree.num_nodes]
        ctx.arbor_allocate(tree, None, self.budget, k)
        ctx.arbor_evict(tree, k)
        return k

    def decode(self):
        """One decode step of every open child: append a token, a9, then a2/a3."""
        ctx, tree = self.sc.ctx, self.tree
        for ch in tree.active:
            self._append(ch)
        q = self.sc.queries(1_000_000 + self.step, len(tree.active))
        self.step += 1
        return q, decode_step(ctx, tree, q)


# ---------------------------------------------------------------- f1: event-driven controller
class Controller:
    """Alg. 2 on the library: every policy update event is one
    ``arbor_policy_event`` call (rehydrate / allocate / evict kernels, no host sync); the
    waterline (Alg. 2 l.31-33, Σ k ≥ 𝓑 − δ, at most one pending Pressure) runs on the device
    (``arbor_policy_waterline``: the check gates a Pressure enqueued behind it)."""

    def __init__(self, ctx: ArborKV, budget: int, delta: int):
        import torch
        self.ctx = ctx
        self.budget = int(budget)
        self.delta = int(delta)
        self.pending = False
        self.k_buf = torch.empty(ctx.max_nodes, dtype=torch.int32, device=ctx.device)
        self.log = []      # (event, node or -1, Σ k after) — read lazily by callers

    def _event(self, tree, kind, node=-1):
        self.ctx.arbor_policy_event(tree, kind, node, self.budget, self.k_buf[:tree.num_nodes])

    def boundary(self, tree, i: int):
        self._event(tree, "boundary", i)
        self.log.append(("boundary", i))

    def transition(self, tree):
        self._event(tree, "transition")
        self.log.append(("transition", -1))

    def pressure(self, tree):
        self._event(tree, "pressure")
        self.pending = False
        self.log.append(("pressure", -1))

    def total(self) -> int:
        return self.ctx.arbor_retained_tokens()

    def waterline(self) -> bool:
        """Host-side waterline (syncs for Σ k): kept for diagnostics; the decode loop uses
        waterline_device."""
        if not self.pending and self.total() >= self.budget - self.delta:
            self.pending = True
            return True
        return False

    def waterline_device(self, tree):
        """Alg. 2 l.31-33 on the device: check M ≥ 𝓑 − δ and, if it fires, Pressure — in one
        call, no host sync (arbor_policy_waterline)."""
        self.ctx.arbor_policy_waterline(tree, self.budget, self.delta, self.k_buf[:tree.num_nodes])
        self.log.append(("waterline", -1))
