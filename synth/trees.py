"""Seeded thought-tree generators (no method arithmetic).

Trees follow the paper's model (§3 Preliminaries): a rooted
tree of thought blocks, node ids dense in creation order (parent id < child
id), each node a contiguous span of one global token stream
(SPEC S:90 design decision).  Shapes follow §5.1 as concretised
in SURVEY.md §8(d).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class SynthTree:
    """A tree snapshot: host arrays in the layout of ``arbor_tree`` (include/arbor.h)."""
    parent: np.ndarray          # int32 [N], -1 for the root
    span_start: np.ndarray      # int64 [N], a_i (absolute position)
    span_len: np.ndarray        # int32 [N], n_i
    is_open: np.ndarray         # uint8 [N]
    v: np.ndarray               # float32 [N] search value v_i in [0,1]
    u: np.ndarray               # float32 [N] uncertainty u_i in [0,1] (Eq. 1)
    active: list = field(default_factory=list)   # active leaves (node ids)

    @property
    def num_nodes(self) -> int:
        return int(self.parent.shape[0])

    @property
    def total_tokens(self) -> int:
        return int(self.span_len.astype(np.int64).sum())

    def copy(self) -> "SynthTree":
        return SynthTree(self.parent.copy(), self.span_start.copy(), self.span_len.copy(),
                         self.is_open.copy(), self.v.copy(), self.u.copy(), list(self.active))

    def add_node(self, parent: int, span_start: int, span_len: int, is_open: bool,
                 v: float, u: float) -> int:
        """Append a node (dense id = current count)."""
        nid = self.num_nodes
        self.parent = np.append(self.parent, np.int32(parent)).astype(np.int32)
        self.span_start = np.append(self.span_start, np.int64(span_start)).astype(np.int64)
        self.span_len = np.append(self.span_len, np.int32(span_len)).astype(np.int32)
        self.is_open = np.append(self.is_open, np.uint8(1 if is_open else 0)).astype(np.uint8)
        self.v = np.append(self.v, np.float32(v)).astype(np.float32)
        self.u = np.append(self.u, np.float32(u)).astype(np.float32)
        return nid

    def end_position(self) -> int:
        """One past the largest absolute position used so far."""
        if self.num_nodes == 0:
            return 0
        return int((self.span_start + self.span_len.astype(np.int64)).max())


def _features(rng: np.random.Generator, n: int):
    v = rng.random(n).astype(np.float32)
    u = rng.random(n).astype(np.float32)
    return v, u


def full_tree(levels: int, width: int, t_node: int, seed: int = 0) -> SynthTree:
    """Complete tree with ``levels`` levels of fan-out ``width``; BFS ids.

    parent(i) = (i-1)//width; spans packed in id order.
    levels counts levels (root = level 1), so full_tree(3,2,32) has 7 nodes
    (BASELINE configs[0]) and full_tree(4,5,128) has 156 (configs[1]).
    """
    n = sum(width ** l for l in range(levels))
    parent = np.array([-1] + [(i - 1) // width for i in range(1, n)], dtype=np.int32)
    span_len = np.full(n, t_node, dtype=np.int32)
    span_start = (np.arange(n, dtype=np.int64) * t_node).astype(np.int64)
    rng = np.random.default_rng(seed)
    v, u = _features(rng, n)
    return SynthTree(parent, span_start, span_len, np.zeros(n, np.uint8), v, u, [])


def search_tree(num_nodes: int, branching: int, max_levels: int, t_node: int,
                seed: int = 0) -> SynthTree:
    """DPTS-like best-first growth (SURVEY §8(d) ``search_tree``).

    First one seeded chain is expanded down to ``max_levels`` levels (each
    chain node gets ``branching`` children); then a frontier leaf with depth
    < max_levels-1 is picked with probability proportional to v and given
    ``branching`` children, the last expansion truncated so that exactly
    ``num_nodes`` nodes exist.
    """
    rng = np.random.default_rng(seed)
    parent = [-1]
    depth = [0]
    v = [float(rng.random())]
    children = {0: []}

    def add(p):
        nid = len(parent)
        parent.append(p)
        depth.append(depth[p] + 1)
        v.append(float(rng.random()))
        children[nid] = []
        children[p].append(nid)
        return nid

    cur = 0
    while depth[cur] < max_levels - 1 and len(parent) < num_nodes:
        kids = []
        for _ in range(branching):
            if len(parent) >= num_nodes:
                break
            kids.append(add(cur))
        if not kids:
            break
        cur = kids[int(rng.integers(len(kids)))]
    while len(parent) < num_nodes:
        frontier = [i for i in range(len(parent))
                    if not children[i] and depth[i] < max_levels - 1]
        if not frontier:
            raise ValueError("search_tree: no expandable frontier left")
        w = np.array([v[i] for i in frontier], dtype=np.float64) + 1e-12
        pick = frontier[int(rng.choice(len(frontier), p=w / w.sum()))]
        for _ in range(branching):
            if len(parent) >= num_nodes:
                break
            add(pick)
    n = len(parent)
    span_len = np.full(n, t_node, dtype=np.int32)
    span_start = (np.arange(n, dtype=np.int64) * t_node).astype(np.int64)
    u = rng.random(n).astype(np.float32)
    return SynthTree(np.array(parent, np.int32), span_start, span_len,
                     np.zeros(n, np.uint8), np.array(v, np.float32), u, [])


def leaves_of(tree: SynthTree) -> list:
    has_child = np.zeros(tree.num_nodes, bool)
    for p in tree.parent:
        if p >= 0:
            has_child[p] = True
    return [i for i in range(tree.num_nodes) if not has_child[i]]


def _depths(parent: np.ndarray) -> np.ndarray:
    d = np.zeros(parent.shape[0], np.int64)
    for i in range(1, parent.shape[0]):
        d[i] = d[parent[i]] + 1
    return d


def highest_v_leaf(tree: SynthTree) -> int:
    """C2's active leaf: the leaf with the highest search value."""
    lv = leaves_of(tree)
    return int(max(lv, key=lambda i: (float(tree.v[i]), -i)))


def dpts_initial_leaves(tree: SynthTree, n_active: int, seed: int) -> list:
    """C3: n_active leaves under distinct level-2 parents (depth-2 nodes)."""
    rng = np.random.default_rng(seed)
    d = _depths(tree.parent)
    lv = leaves_of(tree)
    by_parent = {}
    for leaf in lv:
        if d[leaf] == 3:
            by_parent.setdefault(int(tree.parent[leaf]), []).append(leaf)
    parents = sorted(by_parent)
    if len(parents) < n_active:
        raise ValueError("not enough level-2 parents")
    chosen = rng.choice(len(parents), size=n_active, replace=False)
    return [int(rng.choice(by_parent[parents[c]])) for c in sorted(chosen)]


def dpts_schedule(tree: SynthTree, initial: list, transitions: int, swap: int,
                  seed: int) -> list:
    """C3 transition schedule: each step replaces ``swap`` of the active leaves
    with seeded leaves under currently unused level-2 parents (backtracks into
    possibly evicted subtrees).  Returns a list of active-leaf lists (closed
    leaves of the base tree; the caller opens a child under each)."""
    rng = np.random.default_rng(seed + 7919)
    d = _depths(tree.parent)
    by_parent = {}
    for leaf in leaves_of(tree):
        if d[leaf] == 3:
            by_parent.setdefault(int(tree.parent[leaf]), []).append(leaf)
    cur = list(initial)
    out = []
    for _ in range(transitions):
        used = {int(tree.parent[x]) for x in cur}
        unused = sorted(p for p in by_parent if p not in used)
        drop = sorted(rng.choice(len(cur), size=swap, replace=False).tolist())
        newp = rng.choice(len(unused), size=swap, replace=False).tolist()
        nxt = list(cur)
        for slot, pi in zip(drop, newp):
            nxt[slot] = int(rng.choice(by_parent[unused[pi]]))
        cur = nxt
        out.append(list(cur))
    return out


def tot_expansion(tree: SynthTree, rng: np.random.Generator, width: int, max_depth: int):
    """f1 traces: the next block a Tree-of-Thoughts search expands — a closed node with fewer
    than ``width`` children and depth < ``max_depth``, drawn ∝ v (ties of the draw by id).
    Returns (parent, v, u) of the new child, or None when the tree is complete.  Workload
    generation only (the search policy is outside ArborKV)."""
    d = _depths(tree.parent)
    kids = np.bincount(tree.parent[tree.parent >= 0], minlength=tree.num_nodes)
    elig = [i for i in range(tree.num_nodes)
            if not tree.is_open[i] and kids[i] < width and d[i] < max_depth]
    if not elig:
        return None
    w = np.asarray([float(tree.v[i]) + 1e-3 for i in elig])
    parent = int(elig[int(rng.choice(len(elig), p=w / w.sum()))])
    v, u = _features(rng, 1)
    return parent, float(v[0]), float(u[0])
