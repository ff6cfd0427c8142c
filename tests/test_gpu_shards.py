"""KV-head sharding on one GPU: the multi-GPU path splits the
rows (layer, KV head) across ranks and all-reduces int64 partial node masses.  Here the
"ranks" are contexts over disjoint KV-head ranges on the same device (world size 1 each, so
no NCCL): every shard runs the same arbor_decode_step calls on its slice of the queries, and

* its accumulated attention A equals the full context's rows bit for bit (rows are
  independent: same tiles, same logits, same LSEs, same summation order);
* the shards' partial masses sum (int64, any order) to the full context's Mass exactly —
  the identity the NCCL all-reduce relies on for rank-invariant s, k and page tables;
* s from the summed masses matches the full context's s, and from the same scores every
  shard allocates the same k and evicts to the same page tables and free list.
"""
import math

import numpy as np
import pytest
import torch

import synth
from oracle import msve as omsve, tae as otae
from paper_2605_22106_b200 import workload

from gpu_helpers import oracle_params

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("shards", [2, 4])
def test_head_shards_sum_to_full(shards):
    preset = dict(tree=("full", 3, 4, 96), L=3, H=8, Hq=32, d=128, dtype="bf16", P=16, rho=0.5,
                  params={}, active="highest_v")
    workload.PRESETS["_shard_test"] = preset
    try:
        full = workload.setup("_shard_test", 5)
        hc = preset["H"] // shards
        parts = [workload.setup("_shard_test", 5, kv_head_begin=r * hc, kv_head_count=hc)
                 for r in range(shards)]
    finally:
        del workload.PRESETS["_shard_test"]
    tree = full.tree
    leaves = synth.leaves_of(tree)
    for step in range(12):
        act = [leaves[(5 * step + j) % len(leaves)] for j in range(1 + step % 3)]
        for sc in [full] + parts:
            sc.tree.active = act
            q = sc.queries(step, len(act))
            out = torch.empty_like(q)
            lse = torch.empty((len(act), sc.ctx.L, sc.ctx.Hq), dtype=torch.float32, device="cuda")
            sc.ctx.arbor_decode_step(sc.tree, q, out, lse)
    torch.cuda.synchronize()
    A = full.ctx.score.cpu()
    for r, sc in enumerate(parts):
        assert torch.equal(sc.ctx.score.cpu(), A[:, r * hc:(r + 1) * hc]), f"A rows of shard {r}"
    N = tree.num_nodes
    fs = full.ctx.arbor_read_scores(N)
    ps = [sc.ctx.arbor_read_scores(N) for sc in parts]
    mass = sum(p["mass"] for p in ps)
    mclose = sum(p["mclose"] for p in ps)
    assert np.array_equal(mass, fs["mass"]), "partial masses do not sum to the full Mass"
    assert np.array_equal(mclose, fs["mclose"])
    for p in ps:
        assert np.array_equal(p["nq"], fs["nq"])
    # s from the summed masses (oracle MSVE, the rank-side arithmetic after the all-reduce)
    op = oracle_params(preset["params"])
    s = []
    for i in range(N):
        if tree.is_open[i]:
            s.append(0.5)
            continue
        a = omsve.attention_feature(int(mass[i]), int(mclose[i]), int(fs["nq"][i]), preset["L"],
                                    preset["Hq"])
        s.append(float(np.float32(omsve.msve_score(op["theta"], float(tree.v[i]),
                                                   float(tree.u[i]), a))))
    # the library's fp64 MSVE vs the oracle's: within one f32 ulp (as test_gpu_parity)
    assert np.all(np.abs(np.asarray(s, np.float64) - fs["s"].astype(np.float64)) <= 2.0 ** -23)
    # every rank allocates from the same (all-reduced) scores: identical k on every shard
    B = int(math.floor(preset["rho"] * tree.total_tokens))
    k_full = torch.empty(N, dtype=torch.int32, device="cuda")
    s_dev = torch.as_tensor(fs["s"], device="cuda")
    full.ctx.arbor_allocate(tree, s_dev, B, k_full)
    assert int(k_full.sum()) == B
    for sc in parts:
        k = torch.empty(N, dtype=torch.int32, device="cuda")
        sc.ctx.arbor_allocate(sc.tree, s_dev, B, k)
        assert torch.equal(k, k_full), "rank-side allocation"
    # and the same evictions: page tables and free lists identical across shards
    for sc in [full] + parts:
        sc.ctx.arbor_evict(sc.tree, k_full)
    ref = [full.ctx.arbor_read_node(i) for i in range(N)]
    for sc in parts:
        assert [sc.ctx.arbor_read_node(i) for i in range(N)] == ref, "page tables differ"
        assert sc.ctx.arbor_read_free_list() == full.ctx.arbor_read_free_list()


@pytest.mark.parametrize("shards", [2, 4])
def test_world_size_gt1_external_reduce_bit_identical(shards):
    """The world_size > 1 library path on one device: contexts created as
    ranks r of `shards` (KV-head shards, ARBOR_FLAG_EXTERNAL_REDUCE instead of the NCCL
    communicator, which needs one GPU per rank) run arbor_decode_step with the multi-rank
    finisher (no MSVE in decode_post), the test sums their int64 partial-mass buffers
    (the all-reduce's arithmetic) and each rank runs arbor_score_finish (msve_kernel).
    s, a, k, page tables and free lists must equal the world_size = 1 context's bit for bit,
    step after step, with allocation from the library's own scores (s = NULL)."""
    preset = dict(tree=("full", 3, 4, 96), L=3, H=8, Hq=32, d=128, dtype="bf16", P=16, rho=0.5,
                  params={}, active="highest_v")
    workload.PRESETS["_shard_test"] = preset
    try:
        full = workload.setup("_shard_test", 7)
        hc = preset["H"] // shards
        parts = [workload.setup("_shard_test", 7, kv_head_begin=r * hc, kv_head_count=hc,
                                rank=r, world_size=shards, external_reduce=True)
                 for r in range(shards)]
    finally:
        del workload.PRESETS["_shard_test"]
    tree = full.tree
    N = tree.num_nodes
    leaves = synth.leaves_of(tree)
    B = int(math.floor(preset["rho"] * tree.total_tokens))
    for step in range(6):
        act = [leaves[(7 * step + j) % len(leaves)] for j in range(1 + step % 2)]
        for sc in [full] + parts:
            sc.tree.active = act
            q = sc.queries(step, len(act))
            out = torch.empty_like(q)
            lse = torch.empty((len(act), sc.ctx.L, sc.ctx.Hq), dtype=torch.float32, device="cuda")
            sc.ctx.arbor_decode_step(sc.tree, q, out, lse)
        # the all-reduce: int64 sum of every rank's [Mass | Mclose] partials
        ps = [sc.ctx.arbor_read_scores(N) for sc in parts]
        for sc in parts:
            ptr, cnt = sc.ctx.arbor_mass_buffer()
            assert cnt == 2 * N and ptr != 0
        red = torch.as_tensor(np.concatenate([sum(p["mass"] for p in ps), sum(p["mclose"] for p in ps)]),
                              device="cuda")
        s_parts = []
        for sc in parts:
            s = torch.empty(N, dtype=torch.float32, device="cuda")
            sc.ctx.arbor_score_finish(red, s)
            s_parts.append(s)
        fs = full.ctx.arbor_read_scores(N)
        for sc, s in zip(parts, s_parts):
            r = sc.ctx.arbor_read_scores(N)
            assert np.array_equal(r["mass"], fs["mass"]) and np.array_equal(r["nq"], fs["nq"])
            assert np.array_equal(r["a"].view(np.int32), fs["a"].view(np.int32)), f"a, step {step}"
            assert np.array_equal(r["s"].view(np.int32), fs["s"].view(np.int32)), f"s, step {step}"
            assert np.array_equal(s.cpu().numpy().view(np.int32), fs["s"].view(np.int32))
        if step in (2, 5):
            ks = []
            for sc in [full] + parts:
                k = torch.empty(N, dtype=torch.int32, device="cuda")
                sc.ctx.arbor_allocate(sc.tree, None, B, k)     # the library's own s
                sc.ctx.arbor_evict(sc.tree, k)
                ks.append(k.cpu())
            for k in ks[1:]:
                assert torch.equal(k, ks[0]), f"k differs at step {step}"
            ref = [full.ctx.arbor_read_node(i) for i in range(N)]
            for sc in parts:
                assert [sc.ctx.arbor_read_node(i) for i in range(N)] == ref, "page tables differ"
                assert sc.ctx.arbor_read_free_list() == full.ctx.arbor_read_free_list()
    # finishing without a pending score is a lifecycle error
    with pytest.raises(Exception):
        parts[0].ctx.arbor_score_finish(red)


def test_collective_flag_one_rank_nccl_bit_identical():
    """a10 on hardware with one GPU (ARBOR_FLAG_COLLECTIVE): a one-rank NCCL communicator
    (arbor_nccl_unique_id → ncclCommInitRank) and the multi-rank finisher — partial masses →
    ncclAllReduce(int64, sum) → msve_kernel — on the arbor_decode_step and arbor_score paths.
    Scores, A, k, page tables and free list equal the fused single-rank context's bit for bit;
    NCCL itself (dlopen of libnccl.so.2, init, the collective) runs on the device."""
    from paper_2605_22106_b200.arbor import nccl_unique_id
    preset = dict(tree=("full", 3, 4, 96), L=3, H=8, Hq=32, d=128, dtype="bf16", P=16, rho=0.5,
                  params={}, active="highest_v")
    workload.PRESETS["_coll_test"] = preset
    try:
        ref = workload.setup("_coll_test", 9)
        col = workload.setup("_coll_test", 9, nccl_id=nccl_unique_id(), collective=True)
    finally:
        del workload.PRESETS["_coll_test"]
    tree = ref.tree
    N = tree.num_nodes
    leaves = synth.leaves_of(tree)
    B = int(math.floor(preset["rho"] * tree.total_tokens))
    for step in range(6):
        act = [leaves[(3 * step + j) % len(leaves)] for j in range(1 + step % 2)]
        for sc in (ref, col):
            sc.tree.active = act
            q = sc.queries(step, len(act))
            out = torch.empty_like(q)
            lse = torch.empty((len(act), sc.ctx.L, sc.ctx.Hq), dtype=torch.float32, device="cuda")
            if step % 3 == 2:        # the two-call path: a9, then a2 + a3 (+ a10) in arbor_score
                sc.ctx.arbor_tree_decode_attn(sc.tree, q, out, lse)
                sc.ctx.arbor_score(sc.tree, q, lse)
            else:                    # f2: arbor_decode_step
                sc.ctx.arbor_decode_step(sc.tree, q, out, lse)
        fr, fc = ref.ctx.arbor_read_scores(N), col.ctx.arbor_read_scores(N)
        for key in ("mass", "mclose", "nq"):
            assert np.array_equal(fr[key], fc[key]), (key, step)
        for key in ("a", "s"):
            assert np.array_equal(fr[key].view(np.int32), fc[key].view(np.int32)), (key, step)
        assert torch.equal(ref.ctx.score, col.ctx.score)
        if step in (2, 5):
            ks = []
            for sc in (ref, col):
                k = torch.empty(N, dtype=torch.int32, device="cuda")
                sc.ctx.arbor_allocate(sc.tree, None, B, k)
                sc.ctx.arbor_evict(sc.tree, k)
                ks.append(k.cpu())
            assert torch.equal(ks[0], ks[1]), f"k differs at step {step}"
            assert [ref.ctx.arbor_read_node(i) for i in range(N)] == \
                [col.ctx.arbor_read_node(i) for i in range(N)]
            assert ref.ctx.arbor_read_free_list() == col.ctx.arbor_read_free_list()
