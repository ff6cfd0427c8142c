"""Whole-path oracle state machine (test infrastructure).

Emulates, step by step and on plain Python/numpy data, everything the
library's calls do (include/arbor.h), in the canonical order of SURVEY.md
§8(c).1:
  geometry → score/accumulated attention → node mass +
  MSVE → TAE allocation → evict: select +
  compact (Alg. 1) → stash / lazy rehydration (P:196-199,
  Alg. 2) → tree decode attention.

K/V are never moved here: compaction is token-extractive and rehydration
restores "the same conditioning state as full retention", so the
content of any retained slot is the original K/V at its absolute position.
The oracle therefore tracks, per (row, node), the within-node offset held by
each slot (slot order: DESIGN.md reading Q23*), plus the per-node page lists
and the LIFO free stack of the paged layout (§8(c).1 step 8).
"""
from __future__ import annotations

import math

import numpy as np

from . import attention, geometry, msve, select, tae


class OracleError(Exception):
    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status


ERR_INVALID_ARG, ERR_INFEASIBLE, ERR_INVARIANT, ERR_OUT_OF_PAGES, ERR_STATE = 2, 3, 4, 6, 7


def default_params(**over) -> dict:
    """SURVEY Appendix B defaults (documented choices; the paper gives none)."""
    p = dict(alpha=1.0, gamma=2.0, lambda_d=0.0, lambda_delta=0.5, eta=0.8, r_min=0.05,
             k_min=4, l_tail=8, n_sinks=4, theta=(-1.0, 2.0, 1.0, 4.0),
             alloc_mode=tae.MODE_WATERFILL, select_mode=0, no_rehydrate=False, k_protect=0,
             slice_layers=0, slice_kv_heads=0, select_shared=0)
    p.update(over)
    return p


class ArborOracle:
    """Plain CPU emulation of one rank's ArborKV state.

    K_all, V_all: float64 [L][H][T][d] — the original (stored-dtype-rounded)
    K/V of this rank's rows by absolute position.  num_layers_global and
    num_q_heads_global normalise a_i (Q4)."""

    def __init__(self, K_all, V_all, num_q_heads_local: int, page_size: int, num_pages: int,
                 params: dict, num_layers_global=None, num_q_heads_global=None, layer_begin=0,
                 kv_head_begin=0, num_kv_heads_global=None):
        self.K = np.asarray(K_all, dtype=np.float64)
        self.V = np.asarray(V_all, dtype=np.float64)
        self.L, self.H, self.Tmax, self.d = self.K.shape
        self.Hq = num_q_heads_local
        self.G = self.Hq // self.H
        self.P = page_size
        self.num_pages = num_pages
        self.params = dict(params)
        self.Lg = num_layers_global or self.L
        self.Hqg = num_q_heads_global or self.Hq
        Hg = num_kv_heads_global or (self.Hqg // self.G)
        # thin slice 𝓛 × 𝓗 for a_i (and the shared selection): local rows, and the a_i
        # normalisation |𝓛|·|𝓗_q| (global counts, Q4/Q6)
        sl, sh = int(self.params.get("slice_layers", 0)), int(self.params.get("slice_kv_heads", 0))
        self.slice = msve.slice_rows(self.L, self.H, layer_begin, kv_head_begin, self.Lg, sl, sh)
        self.norm_layers = sl or self.Lg
        self.norm_qheads = (sh * self.G) if sh else self.Hqg
        del Hg
        self.span_start, self.n, self.open = [], [], []
        self.kept = []            # per node: int64 [L][H][k_cur] offset held by each slot
        self.pages = []           # per node: list of live page ids
        self.koff = []            # per node: page-list slot of valid slot 0 (0 <= koff < P, Q23*)
        self.free = list(range(num_pages - 1, -1, -1))   # LIFO, top at the end
        self.A = np.zeros((self.L, self.H, self.Tmax), dtype=np.float64)
        self.Nq, self.Mclose, self.s_last = [], [], []
        self.rehydrations = 0

    # ------------------------------------------------------------ pages
    def _pop(self) -> int:
        if not self.free:
            raise OracleError(ERR_OUT_OF_PAGES, "out of pages")
        return self.free.pop()

    def k_cur(self, i: int) -> int:
        return int(self.kept[i].shape[-1])

    # ------------------------------------------------------------ lifecycle
    def open_node(self, node: int, span_start: int):
        if node != len(self.n):
            raise OracleError(ERR_INVALID_ARG, "node ids are dense")
        self.span_start.append(int(span_start))
        self.n.append(0)
        self.open.append(True)
        self.kept.append(np.zeros((self.L, self.H, 0), dtype=np.int64))
        self.pages.append([])
        self.koff.append(0)
        self.Nq.append(0)
        self.Mclose.append(0)
        self.s_last.append(0.5)          # never scored (Q31)

    def append(self, node: int, ntok: int):
        """Append ntok decoded tokens to an open node: pages are popped in
        token order (§8(c).1 step 8)."""
        if not self.open[node]:
            raise OracleError(ERR_STATE, "append to a closed node")
        new_n = self.n[node] + ntok
        need = -(-new_n // self.P) - len(self.pages[node])
        if need > len(self.free):
            raise OracleError(ERR_OUT_OF_PAGES, "out of pages")
        for _ in range(need):
            self.pages[node].append(self._pop())
        self.n[node] = new_n
        self.kept[node] = np.broadcast_to(np.arange(new_n, dtype=np.int64),
                                          (self.L, self.H, new_n)).copy()

    def node_mass_partial(self, i: int) -> int:
        return msve.node_mass(self.A, self.span_start[i], self.n[i], self.slice)

    def close_node(self, node: int):
        """Boundary: fix n_i, snapshot Mclose_i (Q5), reset Nq_i."""
        if not self.open[node]:
            raise OracleError(ERR_STATE, "closing a closed node")
        if self.n[node] < 1:
            raise OracleError(ERR_INVALID_ARG, "closed nodes need n >= 1")
        self.open[node] = False
        self.Mclose[node] = self.node_mass_partial(node)
        self.Nq[node] = 0

    # ------------------------------------------------------------ geometry
    @staticmethod
    def geometry(tree):
        parent = [int(x) for x in tree.parent]
        d = geometry.depths(parent)
        dist = geometry.delta(parent, tree.active)
        ps = geometry.path_star(parent, tree.active)
        on_path = [i in ps for i in range(len(parent))]
        return d, dist, on_path

    # ------------------------------------------------------------ attention
    def _visible(self, tree, leaf: int, l: int, h: int) -> np.ndarray:
        return attention.visible_positions(tree.parent, leaf, self.span_start,
                                           lambda i: self.kept[i][l, h])

    def decode(self, tree, q):
        """Tree decode attention: q [nA][L][Hq][d] → (o, lse)."""
        q = np.asarray(q, dtype=np.float64)
        nA = len(tree.active)
        o = np.zeros((nA, self.L, self.Hq, self.d))
        lse = np.full((nA, self.L, self.Hq), -np.inf)
        for b, leaf in enumerate(tree.active):
            for l in range(self.L):
                for h in range(self.H):
                    pos = self._visible(tree, leaf, l, h)
                    if pos.size == 0:
                        continue
                    gs = slice(h * self.G, (h + 1) * self.G)
                    ob, lb, _ = attention.attend(q[b, l, gs], self.K[l, h, pos], self.V[l, h, pos])
                    o[b, l, gs] = ob
                    lse[b, l, gs] = lb
        return o, lse

    def score_accumulate(self, tree, q, lse=None):
        """§8(a) a2: A[l][h][t] += Σ_g exp(q·k_t/√d − LSE) over visible t for
        every active leaf, then Nq_i += 1 for closed i on Path(ℓ_b).

        A_i(t) = Σ_{u>b_i} Attn_{u→t}: only queries AFTER block i's end
        count.  The query of an OPEN active leaf ℓ_b is a token of ℓ_b itself
        (it is appended before it attends, Q25), so u ≤ b_{ℓ_b} and ℓ_b's own
        tokens receive nothing; it still attends to them (o, LSE unchanged).
        A closed active leaf's query is the token after it (u > b), which
        counts (reading Q5')."""
        q = np.asarray(q, dtype=np.float64)
        if lse is None:
            _, lse = self.decode(tree, q)
        lse = np.asarray(lse, dtype=np.float64)
        for b, leaf in enumerate(tree.active):
            for l in range(self.L):
                for h in range(self.H):
                    pos = self._visible(tree, leaf, l, h)
                    if pos.size == 0:
                        continue
                    gs = slice(h * self.G, (h + 1) * self.G)
                    p = attention.probabilities(q[b, l, gs], self.K[l, h, pos], lse[b, l, gs])
                    w = p.sum(axis=0)
                    if self.open[leaf]:       # u ≤ b_ℓ: not "later" than its own block
                        a0 = self.span_start[leaf]
                        w = np.where((pos >= a0) & (pos < a0 + self.n[leaf]), 0.0, w)
                    self.A[l, h, pos] += w
            for i in geometry.root_path(tree.parent, leaf):
                if not self.open[i]:
                    self.Nq[i] += 1

    def masses(self) -> list:
        return [self.node_mass_partial(i) if not self.open[i] else 0
                for i in range(len(self.n))]

    def msve(self, tree, masses=None):
        """§8(a) a3: a_i and s_i for every closed node (Q31)."""
        if masses is None:
            masses = self.masses()
        a = [0.0] * len(self.n)
        s = list(self.s_last)
        for i in range(len(self.n)):
            if self.open[i]:
                continue
            a[i] = msve.attention_feature(masses[i], self.Mclose[i], self.Nq[i],
                                          self.norm_layers, self.norm_qheads)
            s[i] = float(np.float32(msve.msve_score(self.params["theta"], float(tree.v[i]),
                                                     float(tree.u[i]), a[i])))
        self.s_last = s
        return a, s

    def score(self, tree, q, lse=None):
        self.score_accumulate(tree, q, lse)
        return self.msve(tree)

    # ------------------------------------------------------------ allocation
    def allocate(self, tree, s, budget: int, mode=None):
        d, dist, on_path = self.geometry(tree)
        mode = self.params["alloc_mode"] if mode is None else mode
        st, k, mf = tae.allocate(mode, s, d, dist, on_path, self.open, self.n, self.params,
                                 budget, parent=[int(x) for x in tree.parent],
                                 leaf=int(tree.active[0]))
        if st != tae.STATUS_OK:
            raise OracleError(ERR_INFEASIBLE, f"infeasible budget, min feasible {mf}")
        return k

    # ------------------------------------------------------------ evict
    def evict(self, tree, k_target, A_f32=None) -> int:
        """Select + compact every non-pinned closed node whose applied target
        k_app = min(k_cur, k_target) drops (Alg. 2 P:567 'evict only if
        k_new < k', Q17), nodes ascending.  A_f32: the f32 accumulated attention that
        orders heavy hitters (default: the oracle's own A rounded to f32).

        Slot layout after eviction (reading Q23*, end-window hole filling): the
        new block is the LAST k_app of the k_cur valid slots, w = k_cur − k_app onward —
        where the block tail 𝒯 (always kept) already sits.  Retained rows inside
        the window stay in place; the i-th hole there (a slot whose row was evicted,
        ascending) receives the i-th retained row from slots < w (ascending).  The window
        starts at page-list slot c = koff + w: the ⌊c/P⌋ leading pages are freed and
        koff ← c mod P (k_app = 0 frees every page, koff ← 0).  The paper fixes only the
        retained set; the slot order is this build's paging choice.  Freed
        pages go on the free stack nodes ascending, each node's run in descending list
        order."""
        if A_f32 is None:
            A_f32 = self.A.astype(np.float32)
        A_f32 = np.asarray(A_f32, np.float32)
        if self.params.get("select_shared", 0):
            # paper-literal shared selection (Q1): one retained set per block, by
            # Â(t) = Σ_{(l,h) ∈ slice} A[l][h][t] (f32 values summed in fp64, rows ascending,
            # rounded to f32), applied to every row
            rows = sorted(self.slice) if self.slice is not None else \
                [(l, h) for l in range(self.L) for h in range(self.H)]
            acc = np.zeros(A_f32.shape[-1], np.float64)
            for (l, h) in rows:
                acc = acc + A_f32[l, h].astype(np.float64)
            A_f32 = np.broadcast_to(acc.astype(np.float32), A_f32.shape)
        _, _, on_path = self.geometry(tree)
        # pinned: open blocks, and Path* unless k_protect or the flattened-stream
        # analogue (its path is a stream, not a protected set) is in force
        path_free = self.params.get("k_protect", 0) or self.params["alloc_mode"] == tae.MODE_STREAM
        evicted = 0
        for j in range(len(self.n)):
            if self.open[j] or (on_path[j] and not path_free):
                continue
            kc = self.k_cur(j)
            k_app = min(kc, max(0, int(k_target[j])))
            if k_app == kc:
                continue
            a, n = self.span_start[j], self.n[j]
            w = kc - k_app                        # first slot of the kept window
            new = np.zeros((self.L, self.H, k_app), dtype=np.int64)
            for l in range(self.L):
                for h in range(self.H):
                    old = [int(x) for x in self.kept[j][l, h]]
                    R = set(select.retained_set(old, n, k_app, self.params["l_tail"],
                                                A_f32[l, h, a:a + n],
                                                self.params.get("select_mode", select.HEAVY),
                                                self.params["n_sinks"],
                                                is_root=int(tree.parent[j]) < 0))
                    holes = [s for s in range(w, kc) if old[s] not in R]
                    movers = [old[s] for s in range(w) if old[s] in R]
                    assert len(holes) == len(movers)
                    row = old[w:kc]
                    for hs, mv in zip(holes, movers):
                        row[hs - w] = mv
                    new[l, h] = row
            self.kept[j] = new
            if k_app > 0:
                c = self.koff[j] + w
                drop = c // self.P
                self.koff[j] = c % self.P
            else:
                drop = len(self.pages[j])
                self.koff[j] = 0
            for p in reversed(self.pages[j][:drop]):
                self.free.append(p)
            self.pages[j] = self.pages[j][drop:]
            evicted += kc - k_app
        return evicted

    # ------------------------------------------------------------ rehydrate
    def rehydrate(self, nodes) -> int:
        """Lazy rehydration (Alg. 2): a node with k_cur < n gets its
        full span back (bit-exact copy of the stash, Q20); full nodes are a no-op and are
        not counted.

        Slot layout (reading Q23r, a paging choice: the paper fixes only that the
        full span is restored).  An evicted closed block's k_cur retained rows fill the last
        k_cur of its n page-list slots (end-window compaction, Q23*, never moves the end);
        its ⌊(n - k_cur)/P⌋ freed leading pages are popped again, nodes ascending, in list
        order, koff ← 0, and every position p goes back to slot p (a full block holds its
        positions in slot order).  Only the n - k_cur evicted rows cross PCIe; the retained
        ones are moved within HBM.  A block evicted to 0 holds no pages: ⌈n/P⌉ are popped.
        """
        nodes = sorted(set(int(x) for x in nodes))
        for i in nodes:
            if self.open[i]:
                raise OracleError(ERR_STATE, "rehydrating an open node")
        if self.params.get("no_rehydrate"):       # f4 ablation: eviction is irreversible
            return 0
        count = 0
        for i in nodes:
            n, kc = self.n[i], self.k_cur(i)
            if kc == n:
                continue
            if kc == 0:                           # no pages left: a fresh list
                lead = -(-n // self.P)
            else:                                 # the freed leading pages of the list
                slots = n - kc - self.koff[i]
                assert slots >= 0 and slots % self.P == 0, "closed block: window ends at slot n"
                lead = slots // self.P
            self.pages[i] = [self._pop() for _ in range(lead)] + self.pages[i]
            self.kept[i] = np.broadcast_to(np.arange(n, dtype=np.int64), (self.L, self.H, n)).copy()
            self.koff[i] = 0
            count += 1
        self.rehydrations += count
        return count

    # ------------------------------------------------------------ views
    def slot_position(self, i: int, l: int, h: int, slot: int) -> int:
        """Within-node offset held by a node's slot (slot < k_cur)."""
        return int(self.kept[i][l, h, slot])

    def page_of_slot(self, i: int, slot: int) -> tuple:
        c = self.koff[i] + slot
        return self.pages[i][c // self.P], c % self.P
