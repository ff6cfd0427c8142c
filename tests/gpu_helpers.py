"""Helpers shared by the GPU parity tests: build the same seeded scenario on both sides
(libarbor through the binding, and the CPU oracle), read the device state back, compare."""
from __future__ import annotations

import numpy as np
import torch

import synth
from oracle.state import ArborOracle, default_params
from oracle import tae

from paper_2605_22106_b200 import workload
from paper_2605_22106_b200.arbor import make_params


def oracle_params(preset_params: dict) -> dict:
    p = default_params()
    p.update(preset_params)
    if isinstance(p.get("alloc_mode"), str):
        p["alloc_mode"] = {"waterfill": 0, "static": 1, "static_drain": 2, "stream": 3}[p["alloc_mode"]]
    if isinstance(p.get("select_mode"), str):
        p["select_mode"] = {"heavy": 0, "tail": 1, "sinks_tail": 2}[p["select_mode"]]
    return p


def rtol_for(dtype: str) -> float:
    """north_star tolerances: 1e-5 relative (fp32), 2e-2 relative (bf16)."""
    return 1e-5 if dtype == "f32" else 2e-2


def rtol_fp32_quantity(dtype: str) -> float:
    """LSE and accumulated attention A are fp32 quantities on both paths: the bf16 path
    multiplies bf16 operands exactly and accumulates, exponentiates and sums in fp32 (only
    the PV operand P is rounded to bf16, which touches the output alone), so they take the
    fp32 tolerance 1e-5 whatever the KV dtype (observed worst
    relative errors ~2e-7 for LSE and ~1.2e-6 for A, profiles/r02_tolerance_report.json)."""
    return 1e-5


# observed errors of every assert_close call, written by conftest to
# gpurun_out/tolerance_report.json at the end of a GPU session
TOL_LOG = []


def assert_close(x, y, rtol, what="", row_frac=1.0):
    """|x − y| ≤ rtol·(|y| + row_frac·max_row|y|), rows = last axis.

    DESIGN.md "Tolerances": attention outputs are weighted sums of V with cancellation, so
    their rounding error scales with the row's magnitude (row_frac = 1: 'relative' per row);
    accumulated attention A is a sum of positive terms, checked elementwise
    (row_frac = 1e-3)."""
    x = np.asarray(x, np.float64)
    y = np.asarray(y, np.float64)
    assert x.shape == y.shape, (what, x.shape, y.shape)
    if y.size == 0:
        return
    finite = np.isfinite(y)
    assert np.array_equal(np.isfinite(x), finite), f"{what}: non-finite mismatch"
    x = np.where(finite, x, 0.0)
    y = np.where(finite, y, 0.0)
    rowmax = np.max(np.abs(y), axis=-1, keepdims=True)
    bound = rtol * (np.abs(y) + rowmax * row_frac)
    err = np.abs(x - y)
    TOL_LOG.append(dict(what=what, rtol=rtol, row_frac=row_frac, n=int(y.size),
                        max_abs_err=float(err.max()),
                        max_err_over_rowmax=float((err / np.maximum(rowmax, 1e-300)).max()),
                        max_rel_err=float((err / np.maximum(np.abs(y), 1e-300)).max()),
                        max_err_over_bound=float((err / np.maximum(bound, 1e-300)).max())))
    bad = err > bound
    if bad.any():
        i = np.argwhere(bad)[0]
        raise AssertionError(f"{what}: {bad.sum()} of {bad.size} outside tolerance; first at "
                             f"{tuple(i)}: got {x[tuple(i)]!r} want {y[tuple(i)]!r}")


class Pair:
    """The same scenario on the GPU (ctx) and in the oracle."""

    def __init__(self, preset: dict, seed: int = 0, tree=None, extra_tokens=0, extra_nodes=0,
                 max_active=16, page_margin=64, params_over=None):
        self.preset = dict(preset)
        self.seed = seed
        self.tree = tree if tree is not None else workload.build_tree(preset, seed)
        p = preset
        T = self.tree.end_position() + extra_tokens
        self.K, self.V, self.E = synth.make_kv(p["L"], p["H"], T, p["d"], p["dtype"], seed,
                                               self.tree.span_start, self.tree.span_len)
        pp = dict(p["params"])
        pp.update(params_over or {})
        self.params_dict = pp
        self.ctx = workload.make_context(p, self.tree, extra_tokens=extra_tokens,
                                         extra_nodes=extra_nodes, max_active=max_active,
                                         params=make_params(**pp), page_margin=page_margin)
        self.Kd, self.Vd = self.K.cuda(), self.V.cuda()
        self.orc = ArborOracle(self.K.double().numpy(), self.V.double().numpy(), p["Hq"],
                               p["P"], self.ctx.NP, oracle_params(pp))
        workload.load_tree(self.ctx, self.tree, self.Kd, self.Vd)
        for i in range(self.tree.num_nodes):
            self.orc.open_node(i, int(self.tree.span_start[i]))
            n = int(self.tree.span_len[i])
            if n:
                self.orc.append(i, n)
            if not self.tree.is_open[i]:
                self.orc.close_node(i)
        self.step = 0
        self.rtol = rtol_for(p["dtype"])
        self.rtol_q = rtol_fp32_quantity(p["dtype"])

    # ------------------------------------------------------------ queries / steps
    def queries(self, n_active: int):
        p = self.preset
        q = synth.make_queries(n_active, p["L"], p["Hq"], p["d"], p["dtype"],
                               workload.query_seed(self.seed, self.step), self.E)
        self.step += 1
        return q

    def decode_both(self, check=True, score=True, fused=False):
        nA = len(self.tree.active)
        q = self.queries(nA)
        qd = q.cuda()
        out = torch.empty_like(qd)
        lse = torch.empty((nA, self.ctx.L, self.ctx.Hq), dtype=torch.float32, device="cuda")
        if fused and score:      # f2: arbor_decode_step (attention + merged score launch)
            self.ctx.arbor_decode_step(self.tree, qd, out, lse)
        else:
            self.ctx.arbor_tree_decode_attn(self.tree, qd, out, lse)
            if score:
                self.ctx.arbor_score(self.tree, qd, lse)
        qn = q.double().numpy()
        o_ref, lse_ref = self.orc.decode(self.tree, qn)
        if score:
            self.orc.score_accumulate(self.tree, qn)
        if check:
            assert_close(out.float().cpu().numpy(), o_ref, self.rtol, "attention output")
            assert_close(lse.cpu().numpy(), lse_ref, self.rtol_q, "LSE", row_frac=0.0)
        return out, lse

    def warmup(self, steps_per_leaf=4, check=False, fused=False):
        saved = list(self.tree.active)
        for leaf in workload.leaf_cycle_order(self.tree, self.seed):
            self.tree.active = [leaf]
            for _ in range(steps_per_leaf):
                self.decode_both(check=check, fused=fused)
        self.tree.active = saved

    # ------------------------------------------------------------ device reads
    def gpu_A(self):
        return self.ctx.score.cpu().numpy()

    def gpu_node(self, node):
        """(k_cur, pages, pos [L][H][k], K rows [L][H][k][d] raw, V rows raw, first_slot):
        the valid slots are first_slot … first_slot + k_cur − 1 of the live page list."""
        kc, n, pages = self.ctx.arbor_read_node(node)
        ko = self.ctx.arbor_read_node_offset(node)
        L, H, P = self.ctx.L, self.ctx.H, self.ctx.P
        if kc == 0:
            return kc, pages, np.zeros((L, H, 0), np.int64), None, None, ko
        idx = torch.as_tensor(pages, device="cuda", dtype=torch.long)
        sl = slice(ko, ko + kc)
        pos = self.ctx.pos_pool[:, idx].permute(0, 2, 1, 3).reshape(L, H, -1)[:, :, sl]
        kr = self.ctx.k_pool[:, idx].permute(0, 2, 1, 3, 4).reshape(L, H, -1, self.ctx.D)[:, :, sl]
        vr = self.ctx.v_pool[:, idx].permute(0, 2, 1, 3, 4).reshape(L, H, -1, self.ctx.D)[:, :, sl]
        return kc, pages, pos.cpu().numpy().astype(np.int64), kr.cpu(), vr.cpu(), ko

    def check_kv_state(self, nodes=None):
        """Bit-exact: k_cur, page lists, pos tags = oracle kept offsets, K/V bytes = original."""
        nodes = range(self.tree.num_nodes) if nodes is None else nodes
        for i in nodes:
            kc, pages, pos, kr, vr, ko = self.gpu_node(i)
            assert kc == self.orc.k_cur(i), (i, kc, self.orc.k_cur(i))
            assert pages == self.orc.pages[i], (i, pages, self.orc.pages[i])
            assert ko == self.orc.koff[i], (i, ko, self.orc.koff[i])
            assert np.array_equal(pos, self.orc.kept[i]), f"kept positions differ at node {i}"
            if kc:
                a = int(self.tree.span_start[i])
                absp = torch.as_tensor(a + pos)
                kref = torch.gather(self.K, 2, absp[..., None].expand(-1, -1, -1, self.ctx.D))
                vref = torch.gather(self.V, 2, absp[..., None].expand(-1, -1, -1, self.ctx.D))
                assert torch.equal(kr.view(torch.int16) if kr.dtype == torch.bfloat16 else kr.view(torch.int32),
                                   kref.view(torch.int16) if kref.dtype == torch.bfloat16 else kref.view(torch.int32)), f"K bytes differ at node {i}"
                assert torch.equal(vr.view(torch.int16) if vr.dtype == torch.bfloat16 else vr.view(torch.int32),
                                   vref.view(torch.int16) if vref.dtype == torch.bfloat16 else vref.view(torch.int32)), f"V bytes differ at node {i}"
        assert self.ctx.arbor_read_free_list() == self.orc.free, "free list differs"

    def discrete_allocate(self, s, budget, mode=None):
        """Oracle allocation on the GPU's own f32 scores (discrete tier (i))."""
        d, dist, on_path = self.orc.geometry(self.tree)
        m = self.orc.params["alloc_mode"] if mode is None else mode
        return tae.allocate(m, [float(x) for x in s], d, dist, on_path, self.orc.open, self.orc.n,
                            self.orc.params, budget, parent=[int(x) for x in self.tree.parent],
                            leaf=int(self.tree.active[0]))
