"""Synthetic Q/K/V of a named head geometry, generated on the device (bench / tools).

Two recipes:
  "iid"        q, k, v ~ N(0, 1) i.i.d. -- no attention structure; the estimator's
               selected lines are scattered (worst case for slash locality).
  "structured" local + heavy-hitter structure, the shape long-context LLM attention
               has (and the shape the reference's own planted generator encodes,
               planted.cpp:33-150):
                 q[i, h] = N(0, 1) + a * u_g + b * w_g
                 k[j, g] = N(0, 1) + a * u_g + c * w_g * [j is a heavy token]
               u_g is a unit direction over all RoPE pairs (after rotation,
               rope(u, i) . rope(u, j) = sum_p |u_p|^2 cos((i - j) theta_p) favours
               small |i - j|: slash lines near the diagonal); w_g lives on the
               lowest-frequency pairs (theta_p * n <= 0.5, position-invariant as in
               planted.cpp:104-111), so heavy tokens attract every query (vertical
               lines).  Heavy tokens: token 0 plus ~1 per 1024, seeded.
Both are seeded and deterministic; values are rounded to the storage dtype.
"""
from __future__ import annotations

import math

import torch


def make_qkv(n: int, hq: int, hkv: int, dim: int = 128, *, kind: str = "structured",
             dtype=torch.bfloat16, seed: int = 0, rope_base: float = 1e7, device="cuda",
             a: float = 2.5, b: float = 2.0, c: float = 12.0, heavy_every: int = 1024):
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    q = torch.empty((n, hq, dim), dtype=dtype, device=device)
    k = torch.empty((n, hkv, dim), dtype=dtype, device=device)
    v = torch.empty((n, hkv, dim), dtype=dtype, device=device)
    step = 1 << 16  # generate in slabs to bound fp32 scratch at large n
    if kind == "iid":
        for t0 in range(0, n, step):
            t1 = min(n, t0 + step)
            q[t0:t1] = torch.randn((t1 - t0, hq, dim), generator=g, device=device).to(dtype)
            k[t0:t1] = torch.randn((t1 - t0, hkv, dim), generator=g, device=device).to(dtype)
            v[t0:t1] = torch.randn((t1 - t0, hkv, dim), generator=g, device=device).to(dtype)
        return q, k, v
    if kind != "structured":
        raise ValueError(kind)
    P = dim // 2
    thetas = torch.tensor([rope_base ** (-2.0 * p / dim) for p in range(P)], device=device)
    low = (thetas * n <= 0.5).nonzero().flatten()
    if low.numel() == 0:
        low = torch.tensor([P - 1], device=device)
    u = torch.randn((hkv, dim), generator=g, device=device)
    u = u / u.norm(dim=-1, keepdim=True)
    w = torch.zeros((hkv, dim), device=device)
    wr = torch.randn((hkv, 2 * low.numel()), generator=g, device=device)
    idx = torch.stack([2 * low, 2 * low + 1], dim=1).flatten()
    w[:, idx] = wr
    w = w / w.norm(dim=-1, keepdim=True)
    group = hq // hkv
    uq = u.repeat_interleave(group, dim=0)
    wq = w.repeat_interleave(group, dim=0)
    nheavy = max(1, n // heavy_every)
    heavy = torch.randint(1, n, (nheavy,), generator=g, device=device)
    heavy = torch.cat([torch.zeros(1, dtype=heavy.dtype, device=device), heavy])
    for t0 in range(0, n, step):
        t1 = min(n, t0 + step)
        m = t1 - t0
        q[t0:t1] = (torch.randn((m, hq, dim), generator=g, device=device) + a * uq + b * wq
                    ).to(dtype)
        k[t0:t1] = (torch.randn((m, hkv, dim), generator=g, device=device) + a * u).to(dtype)
        v[t0:t1] = torch.randn((m, hkv, dim), generator=g, device=device).to(dtype)
    k[heavy] = (k[heavy].float() + c * w).to(dtype)
    return q, k, v


def yarn_temperature(scale: float) -> float:
    """dca.cpp:32-37."""
    if scale <= 1.0:
        return 1.0
    r = 0.1 * math.log(scale) + 1.0
    return 1.0 / (r * r)
