"""Synthetic Q/K/V of a named head geometry, generated on the device (bench / tools).

Recipes:
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
  "planted"    make_planted(): vertical + local-band slash structure strong enough that
               a Vertical-Slash selection captures most of the attention mass (the
               regime the method is for; bench.py's default).
All are seeded and deterministic; values are rounded to the storage dtype.
"""
from __future__ import annotations

import math

import torch


def make_qkv(n: int, hq: int, hkv: int, dim: int = 128, *, kind: str = "planted",
             dtype=torch.bfloat16, seed: int = 0, rope_base: float = 1e7, device="cuda",
             a: float = 2.5, b: float = 2.0, c: float = 12.0, heavy_every: int = 1024):
    if kind == "planted":
        return make_planted(n, hq, hkv, dim, dtype=dtype, seed=seed, rope_base=rope_base,
                            device=device)
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


def make_planted(n: int, hq: int, hkv: int, dim: int = 128, *, dtype=torch.bfloat16,
                 seed: int = 0, rope_base: float = 1e7, device="cuda", local: float = 10.6,
                 band: int = 16384, anchor: float = 4.0, heavy: float = 28.0,
                 heavy_count: int = 64, noise: float = 1.0):
    """Vertical-slash structure at scale, after the reference's planted generator
    (planted.cpp:33-150: a position-invariant shared direction that planted columns key
    on, over unit background noise) plus the local band real long-context attention has:

      q[i, h] = local * u_g + anchor * w_g + noise * N(0, 1)
      k[j, g] = local * u_g + noise * N(0, 1)   (+ heavy * w_g on heavy tokens)

    u_g lives on the RoPE pairs with theta_p in [0.5, 3] / band, so after rotation
    rope(u, i) . rope(u, j) = sum_p |u_p|^2 cos((i - j) theta_p) is ~1 for |i - j| << band
    and averages out beyond it: diagonals near the main one carry ~local^2 / sqrt(D)
    logits (slash lines); w_g lives on the pairs with theta_p * n <= 0.5 (rotation-
    invariant over the whole context), so the heavy tokens (token 0 + heavy_count - 1
    seeded positions per KV head) attract every query with anchor * heavy / sqrt(D)
    logits (vertical lines).  Heads of one KV group share u_g, w_g and the heavy tokens
    and differ by their noise.  Seeded; rounded to the storage dtype."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    P = dim // 2
    thetas = torch.tensor([rope_base ** (-2.0 * p / dim) for p in range(P)], device=device,
                          dtype=torch.float64)
    loc = ((thetas * band >= 0.5) & (thetas * band <= 3.0)).nonzero().flatten()
    inv = (thetas * n <= 0.5).nonzero().flatten()
    if loc.numel() == 0:
        loc = torch.tensor([P // 2], device=device)
    if inv.numel() == 0:
        inv = torch.tensor([P - 1], device=device)

    def on_pairs(pairs):
        x = torch.zeros((hkv, dim), device=device)
        idx = torch.stack([2 * pairs, 2 * pairs + 1], dim=1).flatten()
        x[:, idx] = torch.randn((hkv, idx.numel()), generator=g, device=device)
        return x / x.norm(dim=-1, keepdim=True)

    u, w = on_pairs(loc), on_pairs(inv)
    group = hq // hkv
    uq, wq = u.repeat_interleave(group, dim=0), w.repeat_interleave(group, dim=0)
    q = torch.empty((n, hq, dim), dtype=dtype, device=device)
    k = torch.empty((n, hkv, dim), dtype=dtype, device=device)
    v = torch.empty((n, hkv, dim), dtype=dtype, device=device)
    step = 1 << 16
    for t0 in range(0, n, step):
        t1 = min(n, t0 + step)
        m = t1 - t0
        q[t0:t1] = (local * uq + anchor * wq +
                    noise * torch.randn((m, hq, dim), generator=g, device=device)).to(dtype)
        k[t0:t1] = (local * u + noise * torch.randn((m, hkv, dim), generator=g,
                                                    device=device)).to(dtype)
        v[t0:t1] = torch.randn((m, hkv, dim), generator=g, device=device).to(dtype)
    for gg in range(hkv):
        hv = torch.randint(1, n, (max(0, heavy_count - 1),), generator=g, device=device)
        hv = torch.cat([torch.zeros(1, dtype=hv.dtype, device=device), hv])
        k[hv, gg] = (k[hv, gg].float() + heavy * w[gg]).to(dtype)
    return q, k, v


def yarn_temperature(scale: float) -> float:
    """dca.cpp:32-37."""
    if scale <= 1.0:
        return 1.0
    r = 0.1 * math.log(scale) + 1.0
    return 1.0 / (r * r)
