"""f1 — the event-driven controller on the GPU (arbor_policy_event) against the controller
oracle (oracle/controller.py, Alg. 2), in lockstep on a seeded Tree-of-Thoughts
trace: every Boundary / Transition / Pressure leaves bit-identical k_cur, kept positions,
page lists, K/V bytes, free list and rehydration count (discrete tier: the oracle takes the
GPU's f32 scores and accumulated attention), the waterline fires at the same
steps on both sides, and every decode step's attention output is within tolerance."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import synth
from oracle.controller import ControllerOracle
from paper_2605_22106_b200 import workload

from gpu_helpers import Pair, oracle_params  # noqa: F401

pytestmark = pytest.mark.gpu

T_NODE, WIDTH, DEPTH = 40, 2, 3


def _preset(mode):
    return dict(tree=("full", 1, WIDTH, T_NODE), L=2, H=2, Hq=8, d=128, dtype="bf16", P=16,
                rho=0.5, params=dict(k_min=4, l_tail=4, alloc_mode=mode), active="node3")


@pytest.mark.parametrize("mode,budget,delta", [("waterfill", 180, 16), ("static_drain", 180, 16)])
def test_controller_trace_lockstep(mode, budget, delta):
    expansions = 6
    preset = _preset(mode)
    tree = synth.full_tree(1, WIDTH, T_NODE, 7)
    pr = Pair(preset, seed=7, tree=tree, extra_tokens=T_NODE * (expansions + 1),
              extra_nodes=expansions + 2)
    ctx, orc = pr.ctx, pr.orc
    gctl = workload.Controller(ctx, budget, delta)
    octl = ControllerOracle(orc, budget, delta)
    tree.active = [0]
    rng = np.random.default_rng(11)
    events = {"boundary": 0, "transition": 0, "pressure": 0}

    def scores():
        return [float(x) for x in ctx.arbor_read_scores(tree.num_nodes)["s"]]

    def both(kind, node=-1):
        s, A = scores(), pr.gpu_A()
        if kind == "boundary":
            gctl.boundary(tree, node)
            octl.boundary(tree, node, s, A_f32=A)
        elif kind == "transition":
            gctl.transition(tree)
            octl.transition(tree, s, A_f32=A)
        else:
            gctl.pressure(tree)
            octl.pressure(tree, s, A_f32=A)
        events[kind] += 1
        pr.check_kv_state()
        assert ctx.arbor_read_counters()[0] == orc.rehydrations, f"{kind}: rehydrations differ"
        assert gctl.total() == octl.total(), f"{kind}: retained totals differ"

    def waterline():
        # the device waterline (no host sync): check + gated Pressure in one call; the
        # oracle decides on the host, and the states must agree afterwards
        s, A = scores(), pr.gpu_A()
        p0 = ctx.arbor_pressure_events()
        gctl.waterline_device(tree)
        fired = octl.waterline()
        if fired:
            octl.pressure(tree, s, A_f32=A)
            events["pressure"] += 1
        assert ctx.arbor_pressure_events() - p0 == (1 if fired else 0), "waterline decisions differ"
        pr.check_kv_state()
        assert gctl.total() == octl.total()

    pr.decode_both()
    both("boundary", 0)
    next_pos = int(tree.span_len[0])
    for _ in range(expansions):
        parent, v, u = synth.tot_expansion(tree, rng, WIDTH, DEPTH)
        child = tree.add_node(parent, next_pos, 0, True, v, u)
        ctx.arbor_open_node(child, next_pos)
        orc.open_node(child, next_pos)
        next_pos += T_NODE
        tree.active = [child]
        both("transition")
        waterline()
        for _t in range(T_NODE):
            pos = int(tree.span_start[child]) + int(tree.span_len[child])
            ctx.arbor_append_kv(child, pr.Kd[:, :, pos:pos + 1].contiguous(),
                                pr.Vd[:, :, pos:pos + 1].contiguous())
            orc.append(child, 1)
            tree.span_len[child] += 1
            pr.decode_both()
            waterline()
        ctx.arbor_close_node(child)
        orc.close_node(child)
        tree.is_open[child] = 0
        both("boundary", child)
        waterline()
    assert events["pressure"] > 0 and orc.rehydrations > 0, (events, orc.rehydrations)
    ctx.arbor_sync()


def test_boundary_on_open_block_is_state_error():
    preset = _preset("waterfill")
    tree = synth.full_tree(1, WIDTH, T_NODE, 3)
    pr = Pair(preset, seed=3, tree=tree, extra_tokens=T_NODE, extra_nodes=2)
    child = tree.add_node(0, int(tree.span_len[0]), 0, True, 0.5, 0.5)
    pr.ctx.arbor_open_node(child, int(tree.span_len[0]))
    tree.active = [child]
    k = torch.empty(tree.num_nodes, dtype=torch.int32, device="cuda")
    with pytest.raises(Exception) as e:
        pr.ctx.arbor_policy_event(tree, "boundary", child, 10 ** 6, k)
    assert getattr(e.value, "status", None) == 7
    pr.ctx.arbor_sync()
