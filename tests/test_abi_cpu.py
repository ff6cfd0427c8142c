"""CPU-only checks of the C-ABI boundary: libarbor.so loads without a GPU, exports every
function include/arbor.h declares, and its host-only helpers (tree validation, minimum
feasible budget) agree with the oracle."""
import os
import re
import subprocess

import numpy as np
import pytest

import synth
from oracle import geometry, tae
from oracle.state import default_params

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "arbor.h")


@pytest.fixture(scope="module")
def lib():
    from paper_2605_22106_b200 import build
    build.build()
    from paper_2605_22106_b200 import arbor
    return arbor


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(arbor_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol(lib):
    names = declared_functions()
    assert len(names) >= 25
    out = subprocess.run(["nm", "-D", "--defined-only", lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (arbor_[a-z0-9_]+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    L = lib.load_library()
    for n in names:
        assert hasattr(L, n)
    assert b"sm_100a" in L.arbor_version()


def test_library_targets_sm100a(lib):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib.LIB_PATH],
                         capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in out


def _tree(parent, n, active, is_open=None):
    N = len(parent)
    n = np.asarray(n, np.int32)
    t = synth.SynthTree(np.asarray(parent, np.int32),
                        np.concatenate([[0], np.cumsum(n[:-1])]).astype(np.int64), n,
                        np.asarray(is_open if is_open is not None else [0] * N, np.uint8),
                        np.full(N, 0.5, np.float32), np.full(N, 0.5, np.float32), list(active))
    return t


def test_validate_tree(lib):
    ok = _tree([-1, 0, 0, 1], [4, 4, 4, 4], [3])
    assert lib.validate_tree(ok, 2)[0] == 0
    bad = ok.copy(); bad.parent[2] = 3
    assert lib.validate_tree(bad)[0] == 2
    bad = ok.copy(); bad.span_len[1] = 0
    assert lib.validate_tree(bad)[0] == 2                     # closed node with n = 0
    bad = ok.copy(); bad.span_start[3] = 2
    assert lib.validate_tree(bad)[0] == 2                     # overlaps its parent
    bad = ok.copy(); bad.active = [7]
    assert lib.validate_tree(bad)[0] == 2
    bad = ok.copy(); bad.active = [3, 3]
    assert lib.validate_tree(bad)[0] == 2
    assert lib.validate_tree(ok, 5)[0] == 2                   # n_sinks > n_root
    bad = ok.copy(); bad.is_open[1] = 1
    assert lib.validate_tree(bad)[0] == 2                     # child of an open node
    bad = ok.copy(); bad.v[0] = 1.5
    assert lib.validate_tree(bad)[0] == 2


@pytest.mark.parametrize("mode", ["waterfill", "static", "static_drain"])
def test_min_feasible_budget_matches_oracle(lib, mode):
    rng = np.random.default_rng(0)
    for _ in range(50):
        N = int(rng.integers(1, 60))
        parent = [-1] + [int(rng.integers(0, i)) for i in range(1, N)]
        n = rng.integers(1, 50, size=N)
        active = [int(x) for x in rng.choice(N, size=int(rng.integers(1, min(3, N) + 1)), replace=False)]
        t = _tree(parent, n, active)
        pd = dict(k_min=int(rng.integers(0, 6)), l_tail=int(rng.integers(0, 9)),
                  r_min=float(rng.choice([0.0, 0.05, 0.3])), alloc_mode=mode, n_sinks=0)
        P = lib.make_params(**pd)
        got = lib.min_feasible_budget(P, t)
        op = default_params(**pd)
        op["alloc_mode"] = {"waterfill": 0, "static": 1, "static_drain": 2}[mode]
        d = geometry.depths(parent)
        dist = geometry.delta(parent, active)
        ps = geometry.path_star(parent, active)
        on = [i in ps for i in range(N)]
        # the oracle's answer: smallest B with STATUS_OK
        if mode == "static":
            assert got == 0
            continue
        st, _, mf = tae.allocate(op["alloc_mode"], [0.5] * N, d, dist, on, [0] * N,
                                 [int(x) for x in n], op, -1)
        assert st == tae.STATUS_INFEASIBLE and mf == got
        st, _, _ = tae.allocate(op["alloc_mode"], [0.5] * N, d, dist, on, [0] * N,
                                [int(x) for x in n], op, got)
        assert st == tae.STATUS_OK


def test_no_cpu_fallback_without_gpu(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(lib.ArborError):
        lib.ArborKV(num_layers=1, num_kv_heads=1, num_q_heads=1, head_dim=64, num_pages=4,
                    max_nodes=4, max_node_tokens=8, max_tokens=64, params=lib.make_params())
