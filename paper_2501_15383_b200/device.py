"""Batched device API over the C-ABI: torch CUDA tensors in, torch CUDA tensors out.

Layouts (token-major, as the kernels read them):
    q [n, hq, dim], k / v [n, hkv, dim]  (float32 or bfloat16, contiguous, on cuda)
    out [n, hq, dim] float32, lse [hq, n] float32
    selections: verticals [chunks, hq, cap_v] int32 + nv [chunks, hq], same for slashes.

torch is only the allocator / stream provider here; all compute is in
liblongctx_b200.so (sm_100a).  Nothing in this module has a CPU path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from ._lib import (AttentionInputC, ChunkConfigC, Error, PrefillConfigC, PrefillOutputC,
                   SelectionOptionsC, check, context, lib)

POSITION_MODES = {"standard": 0, "dca_continuous": 1, "dcaContinuous": 1}
PREFILL_MODES = {"full": 0, "sparse": 1}
KERNEL_PATHS = {"auto": 0, "simt": 1, "tc": 2}


@dataclass
class Options:
    force_sink_column: bool = True
    force_local_band: bool = True
    slash_mean: bool = True

    def c(self) -> SelectionOptionsC:
        return SelectionOptionsC(int(self.force_sink_column), int(self.force_local_band),
                                 int(self.slash_mean))


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p()


def _stream(stream=None, ctx=None):
    """The caller's stream, else torch's current stream ON THE CONTEXT'S DEVICE (the C-ABI
    runs every entry on its context's device, whatever device is current)."""
    s = stream if stream is not None else torch.cuda.current_stream(
        ctx.device if ctx is not None else None)
    return C.c_void_p(s.cuda_stream)


def _chunk(cfg):
    if cfg is None:
        return None
    if isinstance(cfg, ChunkConfigC):
        return cfg
    s, c, w = cfg
    return ChunkConfigC(int(s), int(c), int(w))


def _check_tensor(name, t, dtypes=(torch.float32, torch.bfloat16)):
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise Error("cuda", f"{name} must be a CUDA tensor (there is no CPU path)")
    if t.dtype not in dtypes:
        raise Error("config", f"{name} dtype {t.dtype} not in {dtypes}")
    if not t.is_contiguous():
        raise Error("dimension", f"{name} must be contiguous")


def make_input(q, k, v, positions_q=None, positions_k=None, rope_base=1e4, temperature=1.0):
    for nm, t in (("q", q), ("k", k), ("v", v)):
        _check_tensor(nm, t)
    if q.dim() != 3 or k.dim() != 3 or v.dim() != 3:
        raise Error("dimension", "q, k, v must be [n, heads, dim]")
    if not (q.dtype == k.dtype == v.dtype):
        raise Error("config", "q, k, v must share a dtype")
    n, hq, dim = q.shape
    if k.shape != v.shape or k.shape[0] != n or k.shape[2] != dim:
        raise Error("dimension", "attention input matrices must share n and D")
    for p in (positions_q, positions_k):
        if p is not None:
            _check_tensor("positions", p, (torch.int64,))
            if p.numel() != n:
                raise Error("dimension", "positions length must equal row count")
    dt = 0 if q.dtype == torch.float32 else 1
    return AttentionInputC(n, hq, k.shape[1], dim, dt, q.data_ptr(), k.data_ptr(), v.data_ptr(),
                           positions_q.data_ptr() if positions_q is not None else None,
                           positions_k.data_ptr() if positions_k is not None else None,
                           float(rope_base), float(temperature))


def chunked_prefill(q, k, v, *, chunk_len, last_q, budget, mode="sparse",
                    position_mode="standard", dca=None, opts: Options | None = None,
                    positions_q=None, positions_k=None, rope_base=1e4, temperature=1.0,
                    kernel_path="auto", return_selections=True, return_admitted=False,
                    tc_min_entries=0, out=None, lse=None, stream=None, ctx=None, shard=None,
                    return_recall=False, phase="all", est_heads=None, selections=None,
                    record_chunk_events=False, chunks=None):
    """longctx::chunked_prefill (sparse.hpp:125-129) over all heads of one layer.

    shard=(rank, count): KV-line sharding -- out / lse are this shard's partials
    (see lse_scale_partial and paper_2501_15383_b200/shard.py).
    return_recall: the recall check (north star (d)) -- recall [chunks, hq] = mean over
    each chunk's last min(last_q, rows) rows of min(1, exp(lse_sparse - lse_full)).
    phase "select" / "attend" (sharded layers, shard.py): estimator + selection only (for
    query heads est_heads = (h0, h1)), or attention only over the given ``selections``
    (dict verticals / nv / slashes / ns, as returned).  record_chunk_events: per-chunk
    completion events (see stream_wait_chunk).  chunks=(c0, c1): compute chunks [c0, c1)
    only -- the earlier chunks' keys are still prepared, other rows are left untouched."""
    inp = make_input(q, k, v, positions_q, positions_k, rope_base, temperature)
    opts = opts or Options()
    n, hq, dim = q.shape
    dev = q.device
    bv, bs = int(budget[0]), int(budget[1])
    nchunks = max(1, -(-n // max(int(chunk_len), 1)))
    block = min(int(last_q), int(chunk_len))
    cap_v, cap_s = bv + 2, bs + block + 1
    if selections is not None:
        cap_v, cap_s = selections["verticals"].shape[2], selections["slashes"].shape[2]
    if phase == "select":  # no attention: no outputs
        out = lse = torch.empty(0, dtype=torch.float32, device=dev)
    if out is None:
        out = torch.empty((n, hq, dim), dtype=torch.float32, device=dev)
    if lse is None:
        lse = torch.empty((hq, n), dtype=torch.float32, device=dev)
    sel = {}
    sparse = mode == "sparse"
    phases = {"all": 0, "select": 1, "attend": 2}
    if phase not in phases:
        raise Error("config", f"unknown phase {phase}")
    if selections is not None:
        sel = dict(selections)
    elif phase != "all" and not sparse:
        raise Error("config", "select / attend phases apply to sparse prefill")
    elif (return_selections or phase != "all") and sparse:
        sel["verticals"] = torch.zeros((nchunks, hq, cap_v), dtype=torch.int32, device=dev)
        sel["nv"] = torch.zeros((nchunks, hq), dtype=torch.int32, device=dev)
        sel["slashes"] = torch.zeros((nchunks, hq, cap_s), dtype=torch.int32, device=dev)
        sel["ns"] = torch.zeros((nchunks, hq), dtype=torch.int32, device=dev)
    admitted = torch.zeros((nchunks, hq), dtype=torch.int64, device=dev) \
        if return_admitted else None
    recall = torch.zeros((nchunks, hq), dtype=torch.float32, device=dev) \
        if return_recall else None
    pm = POSITION_MODES[position_mode] if isinstance(position_mode, str) else int(position_mode)
    sr, sc = shard if shard is not None else (0, 1)
    eh0, eh1 = est_heads if est_heads is not None else (0, 0)
    cfg = PrefillConfigC(int(chunk_len), int(last_q), bv, bs, PREFILL_MODES[mode], pm,
                         _chunk(dca) or ChunkConfigC(0, 0, 0), opts.c(),
                         KERNEL_PATHS[kernel_path], int(tc_min_entries), int(sr), int(sc),
                         phases[phase], int(eh0), int(eh1), int(bool(record_chunk_events)),
                         *(chunks if chunks is not None else (0, 0)))
    o = PrefillOutputC(out.data_ptr(), lse.data_ptr(),
                       sel["verticals"].data_ptr() if sel else None,
                       sel["nv"].data_ptr() if sel else None,
                       sel["slashes"].data_ptr() if sel else None,
                       sel["ns"].data_ptr() if sel else None, cap_v, cap_s,
                       admitted.data_ptr() if admitted is not None else None,
                       recall.data_ptr() if recall is not None else None)
    ctx = ctx or context(dev.index)
    check(lib().lcx_chunked_prefill(ctx.ptr, C.byref(inp), C.byref(cfg), C.byref(o),
                                    _stream(stream, ctx)))
    res = dict(out=out, lse=lse, **sel)
    if admitted is not None:
        res["admitted"] = admitted
    if recall is not None:
        res["recall"] = recall
    return res


def stream_wait_chunk(chunk, stream, *, device=None, ctx=None):
    """``stream`` waits for chunk ``chunk`` of the last chunked_prefill on the context (run
    with record_chunk_events=True) to have its out / lse rows final."""
    ctx = ctx or context(device)
    check(lib().lcx_stream_wait_chunk(ctx.ptr, int(chunk), C.c_void_p(stream.cuda_stream)))


def estimate_block(q, k, *, q_row0, nq, nk, last_q, position_mode="standard", dca=None,
                   rope_base=1e4, stream=None, ctx=None):
    """est [hq, block, nk] fp32 (sparse.hpp:74-76)."""
    inp = make_input(q, k, k, None, None, rope_base, 1.0)
    hq = q.shape[1]
    block = min(int(last_q), int(nq))
    est = torch.empty((hq, max(block, 1), nk), dtype=torch.float32, device=q.device)
    pm = POSITION_MODES[position_mode]
    d = _chunk(dca)
    ctx = ctx or context(q.device.index)
    check(lib().lcx_estimate_block(ctx.ptr, C.byref(inp), int(q_row0), int(nq), int(nk),
                                   int(last_q), pm, C.byref(d) if d else None, _ptr(est),
                                   _stream(stream, ctx)))
    return est


def line_scores(q, k, *, q_row0, nq, nk, last_q, position_mode="standard", dca=None,
                slash_mean=True, rope_base=1e4, stream=None, ctx=None):
    inp = make_input(q, k, k, None, None, rope_base, 1.0)
    hq = q.shape[1]
    col = torch.empty((hq, nk), dtype=torch.float32, device=q.device)
    sl = torch.empty((hq, nk), dtype=torch.float32, device=q.device)
    d = _chunk(dca)
    ctx = ctx or context(q.device.index)
    check(lib().lcx_line_scores(ctx.ptr, C.byref(inp), int(q_row0), int(nq), int(nk),
                                int(last_q), POSITION_MODES[position_mode],
                                C.byref(d) if d else None, int(slash_mean), _ptr(col), _ptr(sl),
                                _stream(stream, ctx)))
    return col, sl


def select_from_scores(col, slash, *, block, budget, opts: Options | None = None, stream=None,
                       ctx=None):
    opts = opts or Options()
    heads, n = col.shape
    bv, bs = int(budget[0]), int(budget[1])
    cap_v, cap_s = min(bv, n) + 1, min(bs, n) + block
    dev = col.device
    v = torch.zeros((heads, cap_v), dtype=torch.int32, device=dev)
    nv = torch.zeros((heads,), dtype=torch.int32, device=dev)
    s = torch.zeros((heads, cap_s), dtype=torch.int32, device=dev)
    ns = torch.zeros((heads,), dtype=torch.int32, device=dev)
    o = opts.c()
    ctx = ctx or context(dev.index)
    check(lib().lcx_select_from_scores(ctx.ptr, _ptr(col), _ptr(slash), heads, n, int(block), bv,
                                       bs, C.byref(o), _ptr(v), _ptr(nv), cap_v, _ptr(s),
                                       _ptr(ns), cap_s, _stream(stream, ctx)))
    return v, nv, s, ns


def select_critical(est, *, n, budget, opts: Options | None = None, stream=None, ctx=None):
    opts = opts or Options()
    heads, block, nn = est.shape
    if nn != n:
        raise Error("dimension", "estimation block must have n columns")
    bv, bs = int(budget[0]), int(budget[1])
    cap_v, cap_s = min(bv, n) + 1, min(bs, n) + block
    dev = est.device
    v = torch.zeros((heads, cap_v), dtype=torch.int32, device=dev)
    nv = torch.zeros((heads,), dtype=torch.int32, device=dev)
    s = torch.zeros((heads, cap_s), dtype=torch.int32, device=dev)
    ns = torch.zeros((heads,), dtype=torch.int32, device=dev)
    o = opts.c()
    ctx = ctx or context(dev.index)
    check(lib().lcx_select_critical(ctx.ptr, _ptr(est), heads, block, n, bv, bs, C.byref(o),
                                    _ptr(v), _ptr(nv), cap_v, _ptr(s), _ptr(ns), cap_s,
                                    _stream(stream, ctx)))
    return v, nv, s, ns


def sparse_attention(q, k, v, verticals, nv, slashes, ns, *, dca=None, positions_q=None,
                     positions_k=None, rope_base=1e4, temperature=1.0, kernel_path="auto",
                     stream=None, ctx=None):
    inp = make_input(q, k, v, positions_q, positions_k, rope_base, temperature)
    n, hq, dim = q.shape
    out = torch.empty((n, hq, dim), dtype=torch.float32, device=q.device)
    lse = torch.empty((hq, n), dtype=torch.float32, device=q.device)
    d = _chunk(dca)
    ctx = ctx or context(q.device.index)
    check(lib().lcx_sparse_attention(ctx.ptr, C.byref(inp), _ptr(verticals), _ptr(nv),
                                     verticals.shape[-1], _ptr(slashes), _ptr(ns),
                                     slashes.shape[-1], int(d is not None),
                                     C.byref(d) if d else None, KERNEL_PATHS[kernel_path],
                                     _ptr(out), _ptr(lse), _stream(stream, ctx)))
    return out, lse


def full_attention(q, k, v, *, dca=None, positions_q=None, positions_k=None, rope_base=1e4,
                   temperature=1.0, kernel_path="auto", stream=None, ctx=None):
    inp = make_input(q, k, v, positions_q, positions_k, rope_base, temperature)
    n, hq, dim = q.shape
    out = torch.empty((n, hq, dim), dtype=torch.float32, device=q.device)
    lse = torch.empty((hq, n), dtype=torch.float32, device=q.device)
    d = _chunk(dca)
    ctx = ctx or context(q.device.index)
    check(lib().lcx_full_attention(ctx.ptr, C.byref(inp), int(d is not None),
                                   C.byref(d) if d else None, KERNEL_PATHS[kernel_path],
                                   _ptr(out), _ptr(lse), _stream(stream, ctx)))
    return out, lse


def attention_recall(lse_sparse, lse_full, *, slack=1e-5, stream=None, ctx=None):
    """refine.cpp:51-72 with a precision-scaled slack (D3)."""
    _check_tensor("lse_sparse", lse_sparse, (torch.float32,))
    _check_tensor("lse_full", lse_full, (torch.float32,))
    if lse_sparse.numel() != lse_full.numel():
        raise Error("dimension", "recall needs equally many sparse and full lse values")
    n = lse_sparse.numel()
    per = torch.empty(n, dtype=torch.float32, device=lse_sparse.device)
    agg = C.c_double()
    ctx = ctx or context(lse_sparse.device.index)
    check(lib().lcx_attention_recall(ctx.ptr, _ptr(lse_sparse), _ptr(lse_full), n, float(slack),
                                     _ptr(per), C.byref(agg), _stream(stream, ctx)))
    return per, agg.value


def lse_scale_partial(o, lse_own, lse_all, *, stream=None, ctx=None):
    """This shard's half of the KV-line LSE merge: o [n, hq, dim] scaled in place by
    exp(lse_own - lse_tot); returns lse_tot [hq, n] (lse_all [G, hq, n])."""
    _check_tensor("o", o, (torch.float32,))
    _check_tensor("lse_own", lse_own, (torch.float32,))
    _check_tensor("lse_all", lse_all, (torch.float32,))
    n, hq, dim = o.shape
    g = lse_all.shape[0]
    if lse_all.shape[1:] != (hq, n) or lse_own.shape != (hq, n):
        raise Error("dimension", "lse shapes must be [G, hq, n] and [hq, n]")
    tot = torch.empty((hq, n), dtype=torch.float32, device=o.device)
    ctx = ctx or context(o.device.index)
    check(lib().lcx_lse_scale_partial(ctx.ptr, _ptr(o), _ptr(lse_own), _ptr(lse_all), g, n, hq,
                                      dim, _ptr(tot), _stream(stream, ctx)))
    return tot


def lse_merge(o_parts, lse_parts, *, stream=None, ctx=None):
    """Merge G shard partials: o_parts [G, rows, dim], lse_parts [G, rows]."""
    _check_tensor("o_parts", o_parts, (torch.float32,))
    _check_tensor("lse_parts", lse_parts, (torch.float32,))
    g, rows, dim = o_parts.shape
    out = torch.empty((rows, dim), dtype=torch.float32, device=o_parts.device)
    lse = torch.empty((rows,), dtype=torch.float32, device=o_parts.device)
    ctx = ctx or context(o_parts.device.index)
    check(lib().lcx_lse_merge(ctx.ptr, _ptr(o_parts), _ptr(lse_parts), g, rows, dim, _ptr(out),
                              _ptr(lse), _stream(stream, ctx)))
    return out, lse


def chunked_prefill_host(q, k, v, *, chunk_len, last_q, budget, mode="sparse",
                         position_mode="standard", dca=None, opts: Options | None = None,
                         rope_base=1e4, temperature=1.0, kernel_path="auto", out=None, lse=None,
                         return_selections=False, stream=None, ctx=None, device=0, chunks=None):
    """chunked_prefill on HOST tensors (CPU, ideally pinned) through
    lcx_chunked_prefill_host: chunk-pipelined H2D / compute / D2H inside the library.
    Returns host tensors (out [n, hq, dim] fp32, lse [hq, n] fp32, selections)."""
    for nm, t in (("q", q), ("k", k), ("v", v)):
        if not isinstance(t, torch.Tensor) or t.is_cuda:
            raise Error("dimension", f"{nm} must be a host tensor for the host entry")
        if t.dtype not in (torch.float32, torch.bfloat16) or not t.is_contiguous():
            raise Error("config", f"{nm} must be contiguous float32 / bfloat16")
    n, hq, dim = q.shape
    dt = 0 if q.dtype == torch.float32 else 1
    inp = AttentionInputC(n, hq, k.shape[1], dim, dt, q.data_ptr(), k.data_ptr(), v.data_ptr(),
                          None, None, float(rope_base), float(temperature))
    opts = opts or Options()
    bv, bs = int(budget[0]), int(budget[1])
    nchunks = max(1, -(-n // max(int(chunk_len), 1)))
    block = min(int(last_q), int(chunk_len))
    cap_v, cap_s = bv + 2, bs + block + 1
    if out is None:
        out = torch.empty((n, hq, dim), dtype=torch.float32, pin_memory=True)
    if lse is None:
        lse = torch.empty((hq, n), dtype=torch.float32, pin_memory=True)
    sel = {}
    if return_selections and mode == "sparse":
        # page-locked: a copy into pageable memory would block the enqueue of later chunks
        sel["verticals"] = torch.zeros((nchunks, hq, cap_v), dtype=torch.int32, pin_memory=True)
        sel["nv"] = torch.zeros((nchunks, hq), dtype=torch.int32, pin_memory=True)
        sel["slashes"] = torch.zeros((nchunks, hq, cap_s), dtype=torch.int32, pin_memory=True)
        sel["ns"] = torch.zeros((nchunks, hq), dtype=torch.int32, pin_memory=True)
    pm = POSITION_MODES[position_mode] if isinstance(position_mode, str) else int(position_mode)
    cfg = PrefillConfigC(int(chunk_len), int(last_q), bv, bs, PREFILL_MODES[mode], pm,
                         _chunk(dca) or ChunkConfigC(0, 0, 0), opts.c(),
                         KERNEL_PATHS[kernel_path], 0, 0, 1)
    if chunks is not None:
        cfg.chunk_begin, cfg.chunk_end = int(chunks[0]), int(chunks[1])
    o = PrefillOutputC(out.data_ptr(), lse.data_ptr(),
                       sel["verticals"].data_ptr() if sel else None,
                       sel["nv"].data_ptr() if sel else None,
                       sel["slashes"].data_ptr() if sel else None,
                       sel["ns"].data_ptr() if sel else None, cap_v, cap_s, None, None)
    ctx = ctx or context(device)
    with torch.cuda.device(device):
        check(lib().lcx_chunked_prefill_host(ctx.ptr, C.byref(inp), C.byref(cfg), C.byref(o),
                                             _stream(stream, ctx)))
    return dict(out=out, lse=lse, **sel)
