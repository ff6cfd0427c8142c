"""Multi-process (gloo, world size 2, CPU) checks of the sharded path's host logic.

The B200 path shards the KV cache by KV head; every rank computes int64 partial node masses
over its rows and one all-reduce sums them.  Here each rank runs the oracle on
its head shard, all-reduces the partial masses and Mclose with torch.distributed (gloo), and
derives a, s, k — which must equal the single-process result bit for bit.  The query/KV
slicing used by workload.Scenario is checked to hand each rank exactly its heads.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from oracle import msve, tae
from oracle.state import ArborOracle, default_params

PRESET = dict(L=2, H=4, Hq=8, d=64, P=8)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _scenario(h0, hc, seed=0):
    tree = synth.full_tree(3, 3, 24, seed)
    tree.active = [synth.leaves_of(tree)[4]]
    K, V, E = synth.make_kv(PRESET["L"], PRESET["H"], tree.total_tokens, PRESET["d"], "f32", seed,
                            tree.span_start, tree.span_len)
    G = PRESET["Hq"] // PRESET["H"]
    q = synth.make_queries(1, PRESET["L"], PRESET["Hq"], PRESET["d"], "f32", seed + 1, E)
    params = default_params(k_min=2, l_tail=3)
    o = ArborOracle(K[:, h0:h0 + hc].double().numpy(), V[:, h0:h0 + hc].double().numpy(), hc * G,
                    PRESET["P"], 512, params, num_layers_global=PRESET["L"],
                    num_q_heads_global=PRESET["Hq"])
    for i in range(tree.num_nodes):
        o.open_node(i, int(tree.span_start[i]))
        o.append(i, int(tree.span_len[i]))
        o.close_node(i)
    return tree, o, q[:, :, h0 * G:(h0 + hc) * G].double().numpy(), params


def _pipeline(tree, o, q, reduce):
    for _ in range(3):
        o.score_accumulate(tree, q)
    part = np.array(o.masses(), dtype=np.int64)
    mclose = np.array(o.Mclose, dtype=np.int64)
    mass, mcl = reduce(part), reduce(mclose)
    a = [msve.attention_feature(int(mass[i]), int(mcl[i]), o.Nq[i], PRESET["L"], PRESET["Hq"])
         for i in range(tree.num_nodes)]
    s = [float(np.float32(msve.msve_score(o.params["theta"], float(tree.v[i]), float(tree.u[i]), a[i])))
         for i in range(tree.num_nodes)]
    k = o.allocate(tree, s, int(0.4 * tree.total_tokens))
    return mass, s, k


def _worker(rank, ws, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    hc = PRESET["H"] // ws
    tree, o, q, _ = _scenario(rank * hc, hc)

    def reduce(x):
        t = torch.from_numpy(x.copy())
        dist.all_reduce(t)
        return t.numpy()

    mass, s, k = _pipeline(tree, o, q, reduce)
    out[rank] = (mass.tolist(), s, k)
    dist.barrier()
    dist.destroy_process_group()


def test_mass_allreduce_world_size_invariance():
    tree, o, q, _ = _scenario(0, PRESET["H"])
    mass1, s1, k1 = _pipeline(tree, o, q, lambda x: x)
    ws = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(ws, _free_port(), out), nprocs=ws, join=True)
    for r in range(ws):
        mass, s, k = out[r]
        assert mass == mass1.tolist()          # integer masses identical
        assert s == s1                         # identical f32 scores
        assert k == k1                         # identical budgets (→ identical page tables)


def test_query_and_kv_shard_slicing():
    """workload.Scenario draws queries for all heads then slices its KV-head range, so the
    concatenation of every rank's slice equals the single-rank tensor."""
    from paper_2605_22106_b200 import workload
    p = workload.PRESETS["c2"]
    E = torch.randn(2, p["H"], p["d"])
    full = synth.make_queries(1, 2, p["Hq"], p["d"], "bf16", 5, E)
    G = p["Hq"] // p["H"]
    for ws in (2, 4, 8):
        hc = p["H"] // ws
        parts = [full[:, :, r * hc * G:(r + 1) * hc * G] for r in range(ws)]
        assert torch.equal(torch.cat(parts, dim=2), full)
