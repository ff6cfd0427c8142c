"""f3 — Eq. 1 on the device (arbor_boundary_uncertainty) against the oracle's
uncertainty (oracle/msve.py, pinned in test_oracle_pins.py) fed the fp64 softmax of the same
logits: u within 1e-5 (north_star fp32 tolerance; u ∈ [0, 1]) for f32 and bf16 logits, a
Llama-3 vocabulary (128,256) and ragged small ones, masked (−inf) entries, and the closed
forms uniform → 0 and one-hot → 1."""
from __future__ import annotations

import math

import numpy as np
import pytest
import torch

from oracle import msve
from paper_2605_22106_b200 import workload

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    return workload.make_context(workload.PRESETS["c1"], workload.build_tree(workload.PRESETS["c1"], 0))


def _oracle(row: np.ndarray) -> float:
    z = row.astype(np.float64)
    fin = np.isfinite(z)
    m = z[fin].max()
    p = np.zeros_like(z)
    p[fin] = np.exp(z[fin] - m)
    p /= p.sum()
    return msve.uncertainty(list(p[p > 0]), 0.0, int(z.shape[0]))


@pytest.mark.parametrize("vocab,dtype", [(2, torch.float32), (1000, torch.float32),
                                         (128256, torch.float32), (32003, torch.bfloat16),
                                         (128256, torch.bfloat16)])
def test_uncertainty_matches_oracle(ctx, vocab, dtype):
    g = torch.Generator().manual_seed(vocab)
    B = 5
    z = torch.randn((B, vocab), generator=g) * torch.tensor([0.1, 1.0, 3.0, 8.0, 20.0])[:, None]
    z[2, ::7] = -math.inf                                  # masked tokens
    z = z.to(dtype)
    u = torch.empty(B, dtype=torch.float32, device="cuda")
    ctx.arbor_boundary_uncertainty(z.cuda(), u)
    got = u.cpu().numpy()
    want = np.array([_oracle(z[b].float().numpy()) for b in range(B)])
    assert np.all(np.abs(got - want) <= 1e-5), (got, want)


def test_uncertainty_closed_forms(ctx):
    V = 4096
    z = torch.zeros((3, V))
    z[1, :] = -math.inf
    z[1, 17] = 3.0                                         # one-hot → H = 0 → u = 1
    z[2, :] = torch.arange(V, dtype=torch.float32) * 0.0 + 5.0   # uniform → u = 0
    u = torch.empty(3, dtype=torch.float32, device="cuda")
    ctx.arbor_boundary_uncertainty(z.cuda(), u)
    got = u.cpu().numpy()
    assert abs(got[0]) <= 1e-6 and abs(got[1] - 1.0) <= 1e-6 and abs(got[2]) <= 1e-6


def test_theta_fitter_matches_oracle_and_ranks_utility():
    """f3 θ-fitter (arbor_fit_theta) on synthetic hindsight labels: θ and the loss trace
    against the oracle's fp64 fitter (oracle/calibrate.py, same data, same epochs); the
    fitted MSVE scores rank the hidden utility with Spearman ≥ 0.8."""
    import numpy as np
    import torch
    import synth
    from oracle import calibrate as cal
    from paper_2605_22106_b200.arbor import fit_theta
    phi, y, util = synth.hindsight_labels(4000, 3)
    th, (l0, l1) = fit_theta(torch.as_tensor(phi, device="cuda"), torch.as_tensor(y, device="cuda"),
                             epochs=150, lr=4.0)
    th_ref, (r0, r1) = cal.fit_theta([tuple(float(x) for x in p) for p in phi], [float(x) for x in y],
                                     [0.0, 0.0, 0.0, 0.0], 150, 4.0)
    assert abs(l0 - r0) <= 1e-12 * r0 and abs(l1 - r1) <= 1e-9 * r1
    assert np.allclose(th, th_ref, rtol=1e-7, atol=1e-9), (th, th_ref)
    assert l1 < l0
    z = th[0] + phi.astype(np.float64) @ np.asarray(th[1:])
    s = 1.0 / (1.0 + np.exp(-z))
    rs = np.argsort(np.argsort(s))
    ru = np.argsort(np.argsort(util))
    rho = np.corrcoef(rs, ru)[0, 1]
    assert rho >= 0.8, rho
