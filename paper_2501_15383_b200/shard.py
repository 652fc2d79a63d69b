"""Multi-GPU execution of one layer's chunked prefill (north star (e)).

One process per GPU; torch.distributed (NCCL over NVLink / NVSwitch) is the plumbing.
Strategies (``plan``):

  single  G == 1.
  head    KV-head sharding, no collective on the data path: with
          Hkv % G == 0 rank r owns whole KV heads and their query heads.  Selection and
          attention are per query head (D10), so every rank's result is exactly the
          single-GPU result for its heads.
  balanced  (``auto`` at G > 1) the same per-KV-head independence, cut by measured cost:
          the (KV head, chunk) units in KV-head-major order, each costed by one untimed
          calibration run per KV head (per-chunk device times, lcx_get_chunk_ms -- the
          measured chunk costs a DCPP schedule is fitted to, engine_sim.cpp:117-166), are
          split into G contiguous parts of minimal maximum cost; a rank runs each of its
          parts as one chunked prefill over that KV head's query heads and a chunk range
          (whole KV heads in one call).  Rank 0 calibrates and broadcasts the cost table
          (setup only), so every rank derives the same cut; the data path has no collective.
  seq     KV sharding with a log-sum-exp merge (mode "seq", or "auto" when the query heads
          do not split over the ranks by KV group):
            1. sharded estimator: rank r runs the Vertical-Slash estimator + selection of
               every chunk for its head pairs only (lcx phase SELECT, est_head_begin/end);
               a head's lists depend only on its own rows and the keys, so they are
               bitwise the unsharded lists.  One all_reduce (sum of int32 lists, every
               head written by exactly one rank) gives every rank the full selection.
            2. sharded attention: rank r attends, for every row, the KV entries of its
               part of each head's selected lines -- the contiguous part
               [r cnt / G, (r+1) cnt / G) of each sorted vertical and slash list (lcx phase
               ATTEND, shard_rank / shard_count) -- which partitions every row's admitted
               KV entries over the ranks (V∩S and self-fallback ownership follow the full
               lists).
            3. per-chunk merge, overlapped with the next chunks' attention on a side
               stream: once chunk c's partial rows are final (lcx_stream_wait_chunk),
               all_gather of their lse, lcx_lse_scale_partial (o <- o e^(lse_g - lse)),
               reduce_scatter (sum) of the scaled O rows -- rank r ends with rows
               [t0 + r L / G, t0 + (r+1) L / G) of every chunk.

The seq orchestration (``seq_prefill``) is written against torch.distributed with the
device steps injectable, so it runs under world-size-2 gloo on CPU (tests/test_shard.py);
on GPUs the steps are the lcx C-ABI entries.
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
    chunks: tuple | None = None  # head plans: this rank's chunk range [c0, c1) (None = all)
    # balanced plans: this rank's parts [(g0, g1, c0, c1)] -- KV heads [g0, g1) with their
    # query heads over chunks [c0, c1) (None, None = all chunks)
    segments: list | None = None

    def describe(self) -> str:
        if self.kind == "single":
            return "1 GPU"
        if self.segments is not None:
            parts = "; ".join(
                f"KV {a}" + (f"-{b - 1}" if b - a > 1 else "")
                + (f" chunks [{c0}, {c1})" if c0 is not None else "")
                for a, b, c0, c1 in self.segments)
            return (f"cost-balanced head sharding x{self.world} (rank {self.rank}: {parts}; "
                    f"no collective on the data path)")
        if self.kind == "head":
            rng = f", chunks [{self.chunks[0]}, {self.chunks[1]})" if self.chunks else ""
            return (f"head-sharded x{self.world} ({self.hq} Q / {self.hkv} KV heads{rng} on rank "
                    f"{self.rank}; no collective)")
        return (f"KV-sharded x{self.world}: estimator split by head pairs (selections "
                f"all_reduced), each row's KV entries split by line, per-chunk LSE merge "
                f"over NCCL (all_gather lse, reduce_scatter O) overlapped with attention")


def head_partition(hq: int, hkv: int, world: int, split_groups: bool = False):
    """[(h0, h1, g0, g1)] per rank, or None when heads cannot be split evenly by groups.
    Whole KV heads per rank when Hkv % G == 0; with split_groups also G % Hkv == 0, each KV
    head's query heads split over G / Hkv ranks (unbalanced when the group size is not a
    multiple: 7B at G = 8 gives 4 + 3 -- the seq strategy balances that case instead)."""
    group = hq // hkv
    parts = []
    if hkv % world == 0:
        per = hkv // world
        for r in range(world):
            g0 = r * per
            parts.append((g0 * group, (g0 + per) * group, g0, g0 + per))
        return parts
    if split_groups and world % hkv == 0:
        split = world // hkv
        if split > group:
            return None
        for r in range(world):
            g, k = divmod(r, split)
            a, b = g * group + k * group // split, g * group + (k + 1) * group // split
            parts.append((a, b, g, g + 1))
        return parts
    return None


def est_head_ranges(hq: int, hkv: int, world: int):
    """Query-head range [h0, h1) of each rank's share of the estimator: the head PAIRS of
    the tensor-core estimator (one M = 128 tile = two heads of one KV head) split
    contiguously over the ranks (7B: 16 pairs -> 2 per rank at G = 8; 14B: 24 -> 3).
    A rank with no pair gets (0, 0)."""
    group = hq // hkv
    ppg = (group + 1) // 2
    npairs = hkv * ppg

    def first(p):
        return (p // ppg) * group + 2 * (p % ppg)

    def last(p):
        return min(first(p) + 2, (p // ppg) * group + group)

    out = []
    for r in range(world):
        p0, p1 = r * npairs // world, (r + 1) * npairs // world
        out.append((first(p0), last(p1 - 1)) if p1 > p0 else (0, 0))
    return out


def chunk_split(nchunks: int, parts: int, depth_weight: float = 0.063):
    """Contiguous chunk ranges of about equal cost for `parts` ranks sharing a query head.
    Chunk c costs 1 + depth_weight * (c + 1): a constant part (every row admits ~V + S
    entries) plus a part growing with the keys before it (the estimator scores all of them,
    and the far vertical / slash tiles grow with depth); depth_weight fitted to the per-rank
    times of tools/shard_emulate.py at 1M tokens (chunks [0, 17) vs [17, 32): 55 vs 80 ms)."""
    cost = [1.0 + depth_weight * (c + 1) for c in range(nchunks)]
    total = sum(cost)
    bounds, acc, c = [0], 0.0, 0
    for p in range(1, parts):
        target = total * p / parts
        while c < nchunks and acc + cost[c] / 2 <= target:
            acc += cost[c]
            c += 1
        bounds.append(c)
    bounds.append(nchunks)
    return [(bounds[i], bounds[i + 1]) for i in range(parts)]


def plan(n: int, hq: int, hkv: int, world: int, rank: int, mode: str = "auto",
         chunk_len: int = 32768) -> Plan:
    if world == 1:
        return Plan("single", 1, 0, n, hq, hkv, 0, 0, 0, n)
    group = hq // hkv
    if mode in ("auto", "head") and hkv % world != 0 and world % hkv == 0 \
            and group % (world // hkv) != 0:
        # the query heads of a KV head do not divide over its ranks (7B: 7 heads, 2 ranks):
        # every rank takes all of its KV head's query heads and a cost-balanced contiguous
        # range of the chunks -- balanced work, still no collective
        split = world // hkv
        g = rank // split
        nch = -(-n // chunk_len)
        rng = chunk_split(nch, split)[rank % split]
        return Plan("head", world, rank, n, group, 1, g * group, g, 0, n, chunks=rng)
    # auto: head sharding whenever the query heads split over the ranks by KV group (north
    # star (e): "KV-head sharding where heads are at least the GPU count") -- no collective
    # on the data path; KV-line sharding with the LSE merge only when asked (mode "seq") or
    # when the heads do not split
    parts = head_partition(hq, hkv, world, split_groups=True) \
        if mode in ("auto", "head", "head-split") else None
    if parts is not None:
        h0, h1, g0, g1 = parts[rank]
        return Plan("head", world, rank, n, h1 - h0, g1 - g0, h0, g0, 0, n)
    if mode in ("head", "head-split"):
        raise ValueError(f"cannot head-shard {hq}Q/{hkv}KV over {world} ranks")
    rows = n // world
    eh = est_head_ranges(hq, hkv, world)[rank]
    return Plan("seq", world, rank, n, hq, hkv, 0, 0, rank * rows, rows,
                notes={"est_heads": eh})


def balance_units(costs, world: int):
    """Cut the (KV head, chunk) units, KV-head-major, into `world` contiguous non-empty parts
    minimising the largest part's cost (exact: min-max linear partition by dynamic
    programming).  costs [hkv][nchunks].  Returns [(u0, u1)] per rank."""
    import numpy as np
    flat = np.asarray(costs, dtype=np.float64).reshape(-1)
    U = flat.size
    if U < world:
        raise ValueError(f"{U} units cannot feed {world} ranks")
    pre = np.concatenate([[0.0], np.cumsum(flat)])
    # best[i] = min over cuts of the max part cost of units [0, i) in p parts; arg = last cut
    best = pre.copy()
    best[0] = 0.0
    args = []
    for _ in range(1, world):
        nb = np.full(U + 1, np.inf)
        arg = np.zeros(U + 1, dtype=np.int64)
        for i in range(1, U + 1):
            j = np.arange(0, i)
            cand = np.maximum(best[:i], pre[i] - pre[:i])
            cand[0] = np.inf  # every part non-empty
            m = int(np.argmin(cand))
            nb[i], arg[i] = cand[m], j[m]
        best = nb
        args.append(arg)
    cuts = [U]
    i = U
    for arg in reversed(args):
        i = int(arg[i])
        cuts.append(i)
    cuts.append(0)
    cuts = cuts[::-1]
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


def units_to_segments(u0: int, u1: int, nchunks: int):
    """Unit range [u0, u1) (KV-head-major) -> [(g0, g1, c0, c1)], whole KV heads merged into
    one part with (c0, c1) = (None, None)."""
    segs = []
    g = u0 // nchunks
    while g * nchunks < u1:
        c0 = max(0, u0 - g * nchunks)
        c1 = min(nchunks, u1 - g * nchunks)
        if c0 == 0 and c1 == nchunks:
            if segs and segs[-1][2] is None and segs[-1][1] == g:
                segs[-1] = (segs[-1][0], g + 1, None, None)
            else:
                segs.append((g, g + 1, None, None))
        else:
            segs.append((g, g + 1, c0, c1))
        g += 1
    return segs


def balanced_plan(costs, n: int, hq: int, hkv: int, world: int, rank: int) -> Plan:
    """The cost-balanced head plan of `rank` from the per-(KV head, chunk) cost table."""
    nch = len(costs[0])
    u0, u1 = balance_units(costs, world)[rank]
    segs = units_to_segments(u0, u1, nch)
    group = hq // hkv
    g_first, g_last = segs[0][0], segs[-1][1]
    heads = sum((b - a) * group for a, b, _, _ in segs)
    load = float(sum(sum(costs[g][c0 or 0:c1 or nch]) for a, b, c0, c1 in segs
                     for g in range(a, b)))
    return Plan("head", world, rank, n, heads, g_last - g_first, g_first * group, g_first,
                0, n, notes={"group": group, "balanced_cost_ms": load}, segments=segs)


def refine_costs(costs, world: int, measured_ms):
    """One refinement of the balanced cut: every rank's units scaled by that rank's measured
    / predicted time (the per-call overheads a per-KV-head calibration does not see: cold
    chunk ranges, a second call per rank).  Pure and deterministic, so every rank that holds
    the same table and the same gathered times derives the same new cut."""
    nch = len(costs[0])
    out = [list(map(float, r)) for r in costs]
    for r, (u0, u1) in enumerate(balance_units(costs, world)):
        pred = sum(costs[u // nch][u % nch] for u in range(u0, u1))
        f = float(measured_ms[r]) / pred if pred > 0 else 1.0
        for u in range(u0, u1):
            out[u // nch][u % nch] *= f
    return out


def calibrate(q, k, v, ctx, **kw):
    """Per-(KV head, chunk) device ms of this layer: one untimed chunked prefill per KV head
    over its query heads, with per-chunk events (the second of two runs)."""
    n, hq, _ = q.shape
    hkv = k.shape[1]
    group = hq // hkv
    ctx.set_profiling(True)
    costs = []
    for g in range(hkv):
        qg = q[:, g * group:(g + 1) * group].contiguous()
        kg, vg = k[:, g:g + 1].contiguous(), v[:, g:g + 1].contiguous()
        for _ in range(2):
            D.chunked_prefill(qg, kg, vg, return_selections=False, **kw)
        torch.cuda.synchronize()
        costs.append(ctx.chunk_ms())
        del qg, kg, vg
    return costs


def take(p: Plan, q, k, v):
    if p.kind != "head":
        return q, k, v
    if p.segments is not None:
        grp = p.notes["group"]
        return ([q[:, a * grp:b * grp].contiguous() for a, b, _, _ in p.segments],
                [k[:, a:b].contiguous() for a, b, _, _ in p.segments],
                [v[:, a:b].contiguous() for a, b, _, _ in p.segments])
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


def chunk_bounds(n: int, chunk_len: int):
    return [(t0, min(n, t0 + chunk_len)) for t0 in range(0, n, chunk_len)]


def seq_prefill(world, rank, n, chunk_len, est_heads, run_select, run_attend, wait_chunk,
                scale_fn, new_sel, new_out, comm_stream=None, group=None):
    """The seq strategy's orchestration over torch.distributed (see the module doc).

    run_select(h0, h1, sel): fills this rank's heads of the selection log sel (dict of
      [chunks, hq, cap] / [chunks, hq] int32 tensors, zero elsewhere);
    run_attend(sel, out, lse): this rank's partial attention of every chunk (out
      [n, hq, dim] normalised within the shard, lse [hq, n]); enqueued asynchronously;
    wait_chunk(c, stream): stream waits until chunk c's partial rows are final;
    scale_fn(o, lse_own, lse_all) -> lse_tot: the per-shard scaling of the merge.
    Returns (sel, rows [sum_c L_c / G, hq, dim] = this rank's merged rows of every chunk,
    lse_tot [hq, n])."""
    import torch.distributed as dist
    sel = new_sel()
    h0, h1 = est_heads
    if h1 > h0:
        run_select(h0, h1, sel)
    for key in ("verticals", "nv", "slashes", "ns"):  # each head written by one rank
        dist.all_reduce(sel[key], group=group)
    out, lse = new_out()
    run_attend(sel, out, lse)
    hq, dim = out.shape[1], out.shape[2]
    parts, lse_tot = [], torch.empty_like(lse)
    ctx = torch.cuda.stream(comm_stream) if comm_stream is not None else _nullctx()
    with ctx:
        for c, (t0, t1) in enumerate(chunk_bounds(n, chunk_len)):
            wait_chunk(c, comm_stream)
            rows = t1 - t0
            lse_c = lse[:, t0:t1].contiguous()
            lse_all = torch.empty((world, hq, rows), dtype=lse.dtype, device=lse.device)
            dist.all_gather_into_tensor(lse_all.view(-1), lse_c.view(-1), group=group)
            o_c = out[t0:t1]
            lse_tot[:, t0:t1] = scale_fn(o_c, lse_c, lse_all)
            if rows % world == 0:
                mine = torch.empty((rows // world, hq, dim), dtype=out.dtype, device=out.device)
                dist.reduce_scatter_tensor(mine.view(-1), o_c.reshape(-1), group=group)
            else:  # ragged last chunk: all_reduce, keep this rank's slice
                dist.all_reduce(o_c, group=group)
                a, b = rank * rows // world, (rank + 1) * rows // world
                mine = o_c[a:b]
            parts.append(mine)
    if comm_stream is not None:
        torch.cuda.current_stream().wait_stream(comm_stream)
    return sel, torch.cat(parts, dim=0), lse_tot


class _nullctx:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def seq_row_ranges(n: int, chunk_len: int, world: int, rank: int):
    """The global rows [a, b) of each chunk that rank owns after the seq merge."""
    out = []
    for t0, t1 in chunk_bounds(n, chunk_len):
        rows = t1 - t0
        out.append((t0 + rank * rows // world, t0 + (rank + 1) * rows // world))
    return out


def prefill_segments(p: Plan, qs, ks, vs, **kw):
    """A balanced plan's parts, one chunked prefill each (see take()).  Returns
    {"segments": [per-part result]} plus "admitted" / "recall" flattened over the parts'
    own chunks when asked for."""
    from ._lib import context
    res, agg = [], None
    for (a, b, c0, c1), q, k, v in zip(p.segments, qs, ks, vs):
        kw2 = dict(kw, chunks=(c0, c1)) if c0 is not None else kw
        res.append(D.chunked_prefill(q, k, v, **kw2))
        st = context(q.device.index).stats()  # per call: summed over the parts
        agg = st if agg is None else {x: (max if x == "tc_path" else sum)((agg[x], st[x]))
                                      for x in st}
    p.notes["stats"] = agg
    out = {"segments": res}
    for key in ("admitted", "recall"):
        if key in res[0]:
            out[key] = torch.cat([r[key][slice(s[2], s[3])].reshape(-1)
                                  for r, s in zip(res, p.segments)])
    return out


def prefill(p: Plan, q, k, v, **kw):
    if p.segments is not None:
        return prefill_segments(p, q, k, v, **kw)
    if p.kind != "seq":
        if p.chunks is not None:
            kw = dict(kw, chunks=p.chunks)
        return D.chunked_prefill(q, k, v, **kw)
    kw = dict(kw)
    kw.pop("return_selections", None)
    return_admitted = kw.pop("return_admitted", False)
    kw.pop("return_recall", None)
    n, hq, dim = q.shape
    L = int(kw["chunk_len"])
    nch = -(-n // L)
    block = min(int(kw["last_q"]), L)
    bv, bs = kw["budget"]
    cap_v, cap_s = int(bv) + 2, int(bs) + block + 1
    dev = q.device
    res = {}

    def new_sel():
        z = lambda *shape: torch.zeros(shape, dtype=torch.int32, device=dev)  # noqa: E731
        return {"verticals": z(nch, hq, cap_v), "nv": z(nch, hq),
                "slashes": z(nch, hq, cap_s), "ns": z(nch, hq)}

    def new_out():
        return (torch.empty((n, hq, dim), dtype=torch.float32, device=dev),
                torch.empty((hq, n), dtype=torch.float32, device=dev))

    def run_select(h0, h1, sel):
        D.chunked_prefill(q, k, v, phase="select", est_heads=(h0, h1), selections=sel, **kw)

    def run_attend(sel, out, lse):
        r = D.chunked_prefill(q, k, v, phase="attend", selections=sel, shard=(p.rank, p.world),
                              record_chunk_events=True, out=out, lse=lse,
                              return_admitted=return_admitted, **kw)
        if "admitted" in r:
            res["admitted"] = r["admitted"]

    def wait_chunk(c, stream):
        D.stream_wait_chunk(c, stream, device=dev.index)

    comm = p.notes.setdefault("comm_stream", torch.cuda.Stream(device=dev))
    sel, rows, tot = seq_prefill(p.world, p.rank, n, L, p.notes["est_heads"], run_select,
                                 run_attend, wait_chunk, D.lse_scale_partial, new_sel, new_out,
                                 comm_stream=comm)
    res.update(sel)
    res["rows"], res["lse"] = rows, tot
    return res


def e2e(p: Plan, q, k, v, steps, barrier, world, dev, **kw):
    """Same operator through the host-buffer entry: pinned host Q/K/V in, host O / lse /
    selections out, all copies inside the timed region (lcx_chunked_prefill_host; for the
    seq strategy: the rank's Q/K/V copied in, shard.prefill, its merged rows, lse and the
    selection log copied out)."""
    if p.kind == "seq":
        return e2e_seq(p, q, k, v, steps, barrier, world, dev, **kw)
    if p.segments is not None:
        return e2e_segments(p, q, k, v, steps, barrier, world, dev, **kw)
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
    if p.chunks is not None:
        kw["chunks"] = p.chunks
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


def e2e_segments(p: Plan, qs, ks, vs, steps, barrier, world, dev, **kw):
    """e2e of a balanced plan: each part through lcx_chunked_prefill_host from its own
    pinned buffers (the host entry copies only the part's Q rows and the K / V rows up to its
    last chunk), the parts one after another, all inside the timed region."""
    import torch.distributed as dist
    need = sum((q.numel() + k.numel() + v.numel()) * q.element_size() + q.numel() * 4
               + q.shape[1] * q.shape[0] * 4 for q, k, v in zip(qs, ks, vs))
    ok = torch.ones(1, device=dev)
    try:
        import psutil
        if psutil.virtual_memory().available < 1.3 * need * max(1, world):
            ok.zero_()
    except ImportError:
        pass
    if world > 1:
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    if ok.item() == 0:
        return {"value": None, "skipped": "not enough host RAM for every rank's pinned buffers"}
    bufs = []
    for (a, b, c0, c1), q, k, v in zip(p.segments, qs, ks, vs):
        hs = [torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for t in (q, k, v)]
        for h, t in zip(hs, (q, k, v)):
            h.copy_(t)
        n, hq, dim = q.shape
        oh = torch.empty((n, hq, dim), dtype=torch.float32, pin_memory=True)
        lh = torch.empty((hq, n), dtype=torch.float32, pin_memory=True)
        kw2 = dict(kw, chunks=(c0, c1)) if c0 is not None else dict(kw)
        bufs.append((hs, oh, lh, kw2, (c0, c1)))

    def one():
        rs = []
        for hs, oh, lh, kw2, _ in bufs:
            rs.append(D.chunked_prefill_host(*hs, out=oh, lse=lh, return_selections=True,
                                             device=dev.index, **kw2))
        return rs

    one()  # sizes the staging buffers
    barrier()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    t0 = time.perf_counter()
    for _ in range(steps):
        rs = one()
    e1.record(stream)
    barrier()
    wall = (time.perf_counter() - t0) * 1e3
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t[0])
    h2d = d2h = 0
    for (hs, oh, lh, kw2, (c0, c1)), r in zip(bufs, rs):
        n, hq, dim = hs[0].shape
        L = int(kw["chunk_len"])
        a0 = 0 if c0 is None else c0 * L
        a1 = n if c1 is None else min(n, c1 * L)
        h2d += (a1 - a0) * hq * dim * hs[0].element_size() \
            + 2 * a1 * hs[1].shape[1] * dim * hs[1].element_size()
        d2h += (a1 - a0) * hq * (dim + 1) * 4 \
            + sum(r[x][slice(c0, c1)].numel() * 4 for x in ("verticals", "slashes") if x in r) \
            + sum(r[x].numel() * 4 for x in ("nv", "ns") if x in r)
    return {"ms_per_step": ms / steps, "unit": "tokens/s",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "host_wall_ms_per_step": wall / steps,
            "api": "lcx_chunked_prefill_host per part of the balanced plan (pinned host "
                   "buffers, chunk-pipelined copies of the part's rows)"}


def e2e_seq(p: Plan, q, k, v, steps, barrier, world, dev, **kw):
    import torch.distributed as dist
    # every rank pins a full copy of Q / K / V plus its output rows: skip (all ranks alike)
    # rather than drive the host out of memory
    need = (q.numel() + k.numel() + v.numel()) * q.element_size() + q.numel() * 4 // world
    ok = torch.ones(1, device=dev)
    try:
        import psutil
        if psutil.virtual_memory().available < 1.3 * need * world:
            ok.zero_()
    except ImportError:
        pass
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    if ok.item() == 0:
        return {"value": None, "skipped": "not enough host RAM for every rank's pinned buffers"}
    qh = torch.empty(q.shape, dtype=q.dtype, pin_memory=True)
    kh = torch.empty(k.shape, dtype=k.dtype, pin_memory=True)
    vh = torch.empty(v.shape, dtype=v.dtype, pin_memory=True)
    qh.copy_(q)
    kh.copy_(k)
    vh.copy_(v)
    n, hq, dim = q.shape
    qd, kd, vd = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)

    def one():
        for d, h in ((qd, qh), (kd, kh), (vd, vh)):
            d.copy_(h, non_blocking=True)
        r = prefill(p, qd, kd, vd, **kw)
        outs = [r["rows"], r["lse"]] + [r[x] for x in ("verticals", "nv", "slashes", "ns")]
        hs = [torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for t in outs]
        for h, t in zip(hs, outs):
            h.copy_(t, non_blocking=True)
        return hs

    one()
    barrier()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    t0 = time.perf_counter()
    for _ in range(steps):
        hs = one()
    e1.record(stream)
    barrier()
    wall = (time.perf_counter() - t0) * 1e3
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t[0])
    return {"ms_per_step": ms / steps, "unit": "tokens/s",
            "h2d_bytes_per_step": (qh.numel() + kh.numel() + vh.numel()) * qh.element_size(),
            "d2h_bytes_per_step": sum(h.numel() * h.element_size() for h in hs),
            "host_wall_ms_per_step": wall / steps,
            "api": "shard.prefill (seq: sharded estimator, line-sharded attention, NCCL "
                   "LSE merge) between pinned-host copies of this rank's inputs / outputs"}
