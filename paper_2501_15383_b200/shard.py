"""Multi-GPU execution of one layer's chunked prefill (north star (e)).

One process per GPU; torch.distributed (NCCL over NVLink / NVSwitch) is the plumbing.
Strategies (``plan``):

  single  G == 1.
  head    Head sharding, no collective on the data path.  With
          Hkv % G == 0 rank r owns whole KV heads and their query heads (KV-head
          sharding); with G % Hkv == 0 each KV head's query heads are split across
          G / Hkv ranks (e.g. 7B at G = 8: 4 + 3 of the 7 heads of one KV head), each
          rank holding only its KV head.  Selection and attention are per query head
          (D10), so every rank's result is exactly the single-GPU result for its heads.
  seq     KV-line sharding with a log-sum-exp merge: every rank runs the estimator
          and selection for all heads (bitwise-identical lists, no exchange), then
          attends over its contiguous part of each head's sorted vertical / slash lists
          (lcx_prefill_config.shard_rank / shard_count); the partials are merged with
          all_gather(lse) + lcx_lse_scale_partial + reduce_scatter(sum of scaled O), so
          rank r ends with the exact output rows [r n / G, (r+1) n / G).

``merge_partials`` is written against torch.distributed only, so the collective
orchestration is exercised by world-size-2 gloo tests on CPU (tests/test_shard.py) with
the scaling step injected; on GPUs the scaling step is the CUDA kernel.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field

import torch

from . import device as D


@dataclass
class Plan:
    kind: str          # "single" | "head" | "seq"
    world: int
    rank: int
    n: int
    hq: int            # query heads computed on this rank
    hkv: int           # kv heads held by this rank
    h0: int            # first query head
    g0: int            # first kv head
    row0: int = 0      # first output row owned after the merge ("seq")
    rows: int = 0      # output rows owned after the merge
    notes: dict = field(default_factory=dict)

    def describe(self) -> str:
        if self.kind == "single":
            return "1 GPU"
        if self.kind == "head":
            return (f"head-sharded x{self.world} ({self.hq} Q / {self.hkv} KV heads on rank "
                    f"{self.rank}; no collective)")
        return (f"KV-line sharded x{self.world} + LSE merge over NCCL (all_gather lse, "
                f"reduce_scatter O)")


def head_partition(hq: int, hkv: int, world: int):
    """[(h0, h1, g0, g1)] per rank, or None when heads cannot be split evenly by groups."""
    group = hq // hkv
    parts = []
    if hkv % world == 0:
        per = hkv // world
        for r in range(world):
            g0 = r * per
            parts.append((g0 * group, (g0 + per) * group, g0, g0 + per))
        return parts
    if world % hkv == 0:
        split = world // hkv
        if split > group:
            return None
        for r in range(world):
            g, k = divmod(r, split)
            a, b = g * group + k * group // split, g * group + (k + 1) * group // split
            parts.append((a, b, g, g + 1))
        return parts
    return None


def plan(n: int, hq: int, hkv: int, world: int, rank: int, mode: str = "auto") -> Plan:
    if world == 1:
        return Plan("single", 1, 0, n, hq, hkv, 0, 0, 0, n)
    parts = head_partition(hq, hkv, world) if mode in ("auto", "head") else None
    if parts is not None:
        h0, h1, g0, g1 = parts[rank]
        return Plan("head", world, rank, n, h1 - h0, g1 - g0, h0, g0, 0, n)
    if mode == "head":
        raise ValueError(f"cannot head-shard {hq}Q/{hkv}KV over {world} ranks")
    if n % world:
        raise ValueError("seq sharding needs n divisible by the world size")
    rows = n // world
    return Plan("seq", world, rank, n, hq, hkv, 0, 0, rank * rows, rows)


def take(p: Plan, q, k, v):
    if p.kind != "head":
        return q, k, v
    return (q[:, p.h0:p.h0 + p.hq].contiguous(), k[:, p.g0:p.g0 + p.hkv].contiguous(),
            v[:, p.g0:p.g0 + p.hkv].contiguous())


def merge_partials(out, lse, group=None, scale_fn=None):
    """KV-line LSE merge.  out [n, hq, dim] (this shard's normalised partial, scaled in
    place), lse [hq, n].  Returns (rows [n / G, hq, dim] = the exact output rows this rank
    owns, lse_tot [hq, n]).  scale_fn(out, lse, lse_all) -> lse_tot defaults to the CUDA
    kernel lcx_lse_scale_partial."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    n, hq, dim = out.shape
    lse_all = torch.empty((world, hq, n), dtype=lse.dtype, device=lse.device)
    dist.all_gather_into_tensor(lse_all.view(-1), lse.contiguous().view(-1), group=group)
    tot = (scale_fn or D.lse_scale_partial)(out, lse, lse_all)
    rows = torch.empty((n // world, hq, dim), dtype=out.dtype, device=out.device)
    dist.reduce_scatter_tensor(rows.view(-1), out.view(-1), group=group)
    return rows, tot


def prefill(p: Plan, q, k, v, **kw):
    if p.kind != "seq":
        return D.chunked_prefill(q, k, v, **kw)
    r = D.chunked_prefill(q, k, v, shard=(p.rank, p.world), **kw)
    rows, tot = merge_partials(r["out"], r["lse"])
    r["rows"], r["lse"] = rows, tot
    return r


def e2e(p: Plan, q, k, v, steps, barrier, world, dev, **kw):
    """Same operator through the host-buffer entry: pinned host Q/K/V in, host O / lse /
    selections out, all copies inside the timed region (lcx_chunked_prefill_host).
    Head-sharded and single-GPU plans only (the line-sharded merge runs on device)."""
    if p.kind == "seq":
        return {"value": None, "skipped": "e2e host entry covers single / head-sharded plans"}
    try:
        import psutil
        need = (q.numel() + k.numel() + v.numel()) * q.element_size() \
            + q.numel() * 4 + q.shape[1] * q.shape[0] * 4
        if psutil.virtual_memory().available < 1.3 * need * max(1, world):
            return {"value": None, "skipped": "not enough host RAM for pinned buffers"}
    except ImportError:
        pass
    qh = torch.empty(q.shape, dtype=q.dtype, pin_memory=True)
    kh = torch.empty(k.shape, dtype=k.dtype, pin_memory=True)
    vh = torch.empty(v.shape, dtype=v.dtype, pin_memory=True)
    qh.copy_(q)
    kh.copy_(k)
    vh.copy_(v)
    n, hq, dim = q.shape
    oh = torch.empty((n, hq, dim), dtype=torch.float32, pin_memory=True)
    lh = torch.empty((hq, n), dtype=torch.float32, pin_memory=True)
    kw = dict(kw)
    # one untimed call sizes the staging buffers
    D.chunked_prefill_host(qh, kh, vh, out=oh, lse=lh, return_selections=True,
                           device=dev.index, **kw)
    barrier()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    t0 = time.perf_counter()
    for _ in range(steps):
        r = D.chunked_prefill_host(qh, kh, vh, out=oh, lse=lh, return_selections=True,
                                   device=dev.index, **kw)
    e1.record(stream)
    barrier()
    wall = (time.perf_counter() - t0) * 1e3
    ms = e0.elapsed_time(e1)
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t[0])
    sel_bytes = sum(r[x].numel() * 4 for x in ("verticals", "nv", "slashes", "ns") if x in r)
    return {"ms_per_step": ms / steps, "unit": "tokens/s",
            "h2d_bytes_per_step": (qh.numel() + kh.numel() + vh.numel()) * qh.element_size(),
            "d2h_bytes_per_step": oh.numel() * 4 + lh.numel() * 4 + sel_bytes,
            "host_wall_ms_per_step": wall / steps,
            "api": "lcx_chunked_prefill_host (pinned host buffers, chunk-pipelined copies)"}
