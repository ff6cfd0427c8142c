"""Seeded K/V/Q tensors with heavy-hitter and sink structure (no method arithmetic).

Recipe (SURVEY.md §8(d) "K/V"): K, V ~ N(0,1) cast to the storage dtype.
For every row (layer l, KV head h) a unit direction e_{l,h}; per node,
``heavy_per_node`` seeded positions get k += 4e and the root's first
``n_sinks`` positions (the paper's global sinks) get k += 6e.
Queries are q = N(0,1) + 2e for the KV head of the query head's group.
Layout: K, V are [L][H][T][d] by absolute position; Q is [nA][L][Hq][d].
"""
from __future__ import annotations

import numpy as np
import torch


def bf16_round_np(x: np.ndarray) -> np.ndarray:
    """Round float32 -> nearest-even bfloat16, returned as float32 values."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    b = x.view(np.uint32).astype(np.uint64)
    r = ((b + 0x7FFF + ((b >> 16) & 1)) >> 16) << 16
    return (r & 0xFFFFFFFF).astype(np.uint32).view(np.float32)


def heavy_positions(span_start, span_len, heavy_per_node: int, seed: int) -> np.ndarray:
    """Absolute positions that receive the heavy-hitter bump (host, seeded)."""
    rng = np.random.default_rng(seed + 104729)
    out = []
    for a, n in zip(np.asarray(span_start).tolist(), np.asarray(span_len).tolist()):
        if n <= 0:
            continue
        m = min(heavy_per_node, n)
        out.extend((a + rng.choice(n, size=m, replace=False)).tolist())
    return np.array(sorted(out), dtype=np.int64)


def _torch_dtype(dtype: str):
    if dtype in ("f32", "float32"):
        return torch.float32
    if dtype in ("bf16", "bfloat16"):
        return torch.bfloat16
    raise ValueError(dtype)


def make_kv(L: int, H: int, T: int, d: int, dtype: str, seed: int, span_start=None,
            span_len=None, heavy_per_node: int = 4, n_sinks: int = 4, device="cpu"):
    """Return (K, V, E): K,V [L][H][T][d] in ``dtype``; E [L][H][d] float32."""
    g = torch.Generator(device=device).manual_seed(int(seed))
    K = torch.randn((L, H, T, d), generator=g, device=device, dtype=torch.float32)
    V = torch.randn((L, H, T, d), generator=g, device=device, dtype=torch.float32)
    E = torch.randn((L, H, d), generator=g, device=device, dtype=torch.float32)
    E = E / E.norm(dim=-1, keepdim=True)
    if span_start is not None:
        hp = heavy_positions(span_start, span_len, heavy_per_node, seed)
        hp = hp[hp < T]
        if hp.size:
            idx = torch.as_tensor(hp, device=device)
            K[:, :, idx, :] += 4.0 * E[:, :, None, :]
        root_a = int(np.asarray(span_start)[0])
        root_n = int(np.asarray(span_len)[0])
        ns = min(n_sinks, root_n)
        if ns > 0:
            K[:, :, root_a:root_a + ns, :] += 6.0 * E[:, :, None, :]
    td = _torch_dtype(dtype)
    return K.to(td).contiguous(), V.to(td).contiguous(), E


def make_queries(n_active: int, L: int, Hq: int, d: int, dtype: str, seed: int, E,
                 device="cpu"):
    """q = N(0,1) + 2 e_{l, g // G}; shape [nA][L][Hq][d] in ``dtype``."""
    H = E.shape[1]
    G = Hq // H
    g = torch.Generator(device=device).manual_seed(int(seed) + 12345)
    q = torch.randn((n_active, L, Hq, d), generator=g, device=device, dtype=torch.float32)
    e = E.to(device).repeat_interleave(G, dim=1)          # [L][Hq][d]
    q = q + 2.0 * e[None]
    return q.to(_torch_dtype(dtype)).contiguous()


def hindsight_labels(n: int, seed: int, noise: float = 0.05):
    """Synthetic stand-ins for MSVE calibration labels (the paper's are leave-one-out
    accuracy drops, which need models): features φ = (v, u, a) ~ U(0,1)³ and a
    hidden utility y = clip(0.55 v + 0.15 u + 0.30 a + N(0, noise²), 0, 1).  Returns
    (phi float32 [n][3], y float32 [n], utility without noise float64 [n])."""
    rng = np.random.default_rng(seed)
    phi = rng.random((n, 3))
    util = 0.55 * phi[:, 0] + 0.15 * phi[:, 1] + 0.30 * phi[:, 2]
    y = np.clip(util + rng.normal(0.0, noise, n), 0.0, 1.0)
    return phi.astype(np.float32), y.astype(np.float32), util
