"""MSVE θ calibration (oracle, test infrastructure) — SURVEY §8(f) f3 "the MSVE θ-fitter on
synthetic hindsight labels".

PAPER.md §5.1: θ is "calibrated offline using hindsight interventions on
full-retention trajectories" — each closed block's cache is masked and the normalised
accuracy drop is the supervision signal for optimising θ.  The paper gives no loss or
optimiser; SPEC fixes one, adopted here:
  loss  L(θ) = mean_i (σ(θᵀx_i) − y_i)², x_i = (1, v_i, u_i, a_i)   (MSE on σ)
  step  full-batch gradient descent, ∇_k L = mean_i 2(σ_i − y_i) σ_i (1 − σ_i) x_ik;
        a step that would raise the loss halves the rate and retries (at most 20 halvings;
        the reduced rate is kept), so the loss never increases.
Real hindsight labels need models and datasets (OUT); the tests use synthetic
labels from a hidden θ*.  Parity of the θ *values* stays unpinned.
fp64, plain loops over the examples in index order.
"""
from __future__ import annotations

import math


def sigmoid(z: float) -> float:
    return 1.0 / (1.0 + math.exp(-z))


def loss(theta, phi, y) -> float:
    """L(θ) = mean (σ(θ₀ + θ_v v + θ_u u + θ_a a) − y)²."""
    tot = 0.0
    for (v, u, a), t in zip(phi, y):
        z = theta[0] + theta[1] * v + theta[2] * u + theta[3] * a
        d = sigmoid(z) - t
        tot += d * d
    return tot / len(y)


def grad(theta, phi, y):
    g = [0.0, 0.0, 0.0, 0.0]
    for (v, u, a), t in zip(phi, y):
        z = theta[0] + theta[1] * v + theta[2] * u + theta[3] * a
        s = sigmoid(z)
        c = 2.0 * (s - t) * s * (1.0 - s)
        for k, x in enumerate((1.0, v, u, a)):
            g[k] += c * x
    return [x / len(y) for x in g]


def fit_theta(phi, y, theta0, epochs: int, lr: float):
    """Full-batch GD with loss-nonincrease backoff.  Returns (θ, [initial loss, final loss])."""
    if len(y) < 1:
        raise ValueError("empty example set")
    theta = [float(x) for x in theta0]
    cur = loss(theta, phi, y)
    first = cur
    for _ in range(epochs):
        g = grad(theta, phi, y)
        step = lr
        accepted = False
        for _ in range(21):               # the step, then up to 20 halvings
            cand = [theta[k] - step * g[k] for k in range(4)]
            lc = loss(cand, phi, y)
            if lc <= cur:
                accepted = True
                break
            step *= 0.5
        if not accepted:
            break
        theta, cur, lr = cand, lc, step
    return theta, [first, cur]
