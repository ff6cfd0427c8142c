"""Tree geometry (oracle, test infrastructure).

PAPER.md §3 Preliminaries: rooted tree T=(V,E); d_i = depth (root at
depth 0); Δ_i = shortest-path distance in T from i to the active leaf ℓ*;
Path* = the ancestor chain root→ℓ*.  Several active leaves (DPTS frontier,
P:281) are read per SURVEY Q14: Path* = union of chains, Δ_i = min distance.
"""
from __future__ import annotations

from collections import deque


def depths(parent) -> list:
    """d_root = 0, d_child = d_parent + 1."""
    parent = [int(p) for p in parent]
    d = [0] * len(parent)
    for i, p in enumerate(parent):
        if p >= 0:
            if p >= i:
                raise ValueError("parent id must be < child id")
            d[i] = d[p] + 1
    return d


def root_path(parent, leaf: int) -> list:
    """Path(ℓ): the chain from the root to ℓ, inclusive, root first."""
    out = []
    x = int(leaf)
    while x >= 0:
        out.append(x)
        x = int(parent[x])
    return out[::-1]


def path_star(parent, active) -> set:
    """Path* = ∪_{ℓ ∈ active} Path(ℓ) (Q14)."""
    s = set()
    for leaf in active:
        s.update(root_path(parent, leaf))
    return s


def tree_distance(parent, i: int, j: int) -> int:
    """dist(i,j) = d_i + d_j − 2·d_lca(i,j), the unique tree metric."""
    pi = root_path(parent, i)
    pj = root_path(parent, j)
    common = 0
    for a, b in zip(pi, pj):
        if a != b:
            break
        common += 1
    # lca depth = common - 1; d_i = len(pi) - 1
    return (len(pi) - 1) + (len(pj) - 1) - 2 * (common - 1)


def delta(parent, active) -> list:
    """Δ_i = min_{ℓ ∈ active} dist(i, ℓ) (Alg. 2 P:565 TreeDistance)."""
    n = len(parent)
    if not active:
        raise ValueError("at least one active leaf is required")
    return [min(tree_distance(parent, i, leaf) for leaf in active) for i in range(n)]


def bfs_distances(parent, src: int) -> list:
    """Breadth-first search on the undirected tree (cross-check)."""
    n = len(parent)
    adj = [[] for _ in range(n)]
    for i, p in enumerate(parent):
        if p >= 0:
            adj[i].append(int(p))
            adj[int(p)].append(i)
    dist = [-1] * n
    dist[src] = 0
    dq = deque([src])
    while dq:
        x = dq.popleft()
        for y in adj[x]:
            if dist[y] < 0:
                dist[y] = dist[x] + 1
                dq.append(y)
    return dist


def pinned(parent, active, is_open) -> list:
    """Pinned = Path* ∪ {open nodes} (invariant (i) P:104 read as k_i = n_i,
    Q19; open blocks are not yet eligible for eviction, P:124 'closed block')."""
    ps = path_star(parent, active)
    return [(i in ps) or bool(is_open[i]) for i in range(len(parent))]
