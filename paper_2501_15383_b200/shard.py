"""Multi-GPU execution of one layer's chunked prefill (north star (e)).

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch for the plumbing).
Two strategies, chosen by ``plan``:

  head   KV-head sharding (Hkv % G == 0): rank r owns KV heads [r Hkv/G, (r+1) Hkv/G)
         and their Hq/Hkv query heads; selection, attention and outputs are
         head-local, so there is NO collective on the data path.
  single G == 1.

The KV-sequence / line-sharded strategy with the log-sum-exp merge lives in
``shard_seq`` (added with the per-chunk session API).
"""
from __future__ import annotations

import time
from dataclasses import dataclass

import torch

from . import device as D


@dataclass
class Plan:
    kind: str          # "single" | "head"
    world: int
    rank: int
    n: int
    hq: int            # query heads on this rank
    hkv: int           # kv heads on this rank
    h0: int            # first query head
    g0: int            # first kv head
    row0: int = 0

    def describe(self) -> str:
        if self.kind == "single":
            return "1 GPU"
        return f"KV-head sharded x{self.world} ({self.hkv} KV / {self.hq} Q heads per GPU)"


def plan(n: int, hq: int, hkv: int, world: int, rank: int, mode: str = "auto") -> Plan:
    if world == 1:
        return Plan("single", 1, 0, n, hq, hkv, 0, 0)
    if mode in ("auto", "head") and hkv % world == 0:
        kv = hkv // world
        grp = hq // hkv
        return Plan("head", world, rank, n, kv * grp, kv, rank * kv * grp, rank * kv)
    raise NotImplementedError(
        f"KV-head sharding needs Hkv % G == 0 (Hkv={hkv}, G={world}); "
        "the line-sharded strategy is selected with mode='seq'")


def take(p: Plan, q, k, v):
    if p.kind == "single":
        return q, k, v
    return (q[:, p.h0:p.h0 + p.hq].contiguous(), k[:, p.g0:p.g0 + p.hkv].contiguous(),
            v[:, p.g0:p.g0 + p.hkv].contiguous())


def prefill(p: Plan, q, k, v, **kw):
    return D.chunked_prefill(q, k, v, **kw)


def e2e(p: Plan, q, k, v, steps, barrier, world, dev, **kw):
    """Same operator through the host-buffer entry: pinned host Q/K/V in, host O / lse /
    selections out, all copies inside the timed region (lcx_chunked_prefill_host)."""
    try:
        import psutil
        need = (q.numel() + k.numel() + v.numel()) * q.element_size() \
            + q.numel() * 4 + q.shape[1] * q.shape[0] * 4
        if psutil.virtual_memory().available < 1.3 * need:
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
