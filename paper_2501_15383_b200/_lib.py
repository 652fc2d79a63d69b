"""ctypes binding of the C-ABI in include/longctx_b200.h (liblongctx_b200.so).

The shared library is built in-tree (``python -m paper_2501_15383_b200.build``) and is
the ONLY compute path: there is no CPU fallback.  Loading fails loudly when the
library is missing, and every compute entry fails with kind "cuda" without an
sm_100 device.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "liblongctx_b200.so")

KINDS = {1: "dimension", 2: "config", 3: "domain", 4: "causality", 5: "empty_row",
         6: "empty_calibration", 100: "cuda", 101: "internal"}


class Error(Exception):
    """Mirror of longctx::Error (errors.hpp:12-39): a stable machine-readable kind."""

    def __init__(self, kind: str, message: str):
        super().__init__(message)
        self.kind = kind
        self.message = message

    def __str__(self):
        return f"{self.kind}: {self.message}"


class ChunkConfigC(C.Structure):
    _fields_ = [("chunk_size", C.c_int64), ("train_len", C.c_int64),
                ("local_window", C.c_int64)]


class SelectionOptionsC(C.Structure):
    _fields_ = [("force_sink_column", C.c_int32), ("force_local_band", C.c_int32),
                ("slash_mean", C.c_int32)]


class AttentionInputC(C.Structure):
    _fields_ = [("n", C.c_int64), ("hq", C.c_int32), ("hkv", C.c_int32), ("dim", C.c_int32),
                ("dtype", C.c_int32), ("q", C.c_void_p), ("k", C.c_void_p), ("v", C.c_void_p),
                ("positions_q", C.c_void_p), ("positions_k", C.c_void_p),
                ("rope_base", C.c_double), ("temperature", C.c_double)]


class PrefillConfigC(C.Structure):
    _fields_ = [("chunk_len", C.c_int64), ("last_q", C.c_int64),
                ("budget_vertical", C.c_int64), ("budget_slash", C.c_int64),
                ("mode", C.c_int32), ("position_mode", C.c_int32), ("dca", ChunkConfigC),
                ("opts", SelectionOptionsC), ("kernel_path", C.c_int32),
                ("tc_min_entries", C.c_int32), ("shard_rank", C.c_int32),
                ("shard_count", C.c_int32), ("phase", C.c_int32),
                ("est_head_begin", C.c_int32), ("est_head_end", C.c_int32),
                ("record_chunk_events", C.c_int32), ("chunk_begin", C.c_int32),
                ("chunk_end", C.c_int32)]


class PrefillOutputC(C.Structure):
    _fields_ = [("out", C.c_void_p), ("lse", C.c_void_p), ("sel_verticals", C.c_void_p),
                ("sel_nv", C.c_void_p), ("sel_slashes", C.c_void_p), ("sel_ns", C.c_void_p),
                ("cap_v", C.c_int64), ("cap_s", C.c_int64), ("admitted", C.c_void_p),
                ("recall", C.c_void_p)]


class PrefillStatsC(C.Structure):
    _fields_ = [("chunks", C.c_int64), ("launches", C.c_int64), ("tc_tiles", C.c_int64),
                ("simt_entries", C.c_int64), ("ms_estimate", C.c_double),
                ("ms_select", C.c_double), ("ms_attention", C.c_double),
                ("ms_tc_kernel", C.c_double), ("ms_total", C.c_double),
                ("tc_path", C.c_int64)]


EXPORTS = [
    "lcx_context_create", "lcx_context_destroy", "lcx_last_error", "lcx_version",
    "lcx_device_ok", "lcx_set_profiling", "lcx_get_stats", "lcx_estimate_block",
    "lcx_line_scores", "lcx_select_from_scores", "lcx_select_critical", "lcx_sparse_attention",
    "lcx_full_attention", "lcx_chunked_prefill", "lcx_chunked_prefill_host",
    "lcx_attention_recall", "lcx_lse_merge", "lcx_lse_scale_partial", "lcx_attention_rel",
    "lcx_stream_wait_chunk", "lcx_get_chunk_ms",
]

_lib = None
_lock = threading.Lock()


def lib() -> C.CDLL:
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise Error("cuda", f"{LIB_PATH} is not built (python -m "
                                    "paper_2501_15383_b200.build); there is no CPU fallback")
            L = C.CDLL(LIB_PATH)
            L.lcx_last_error.restype = C.c_char_p
            L.lcx_version.restype = C.c_char_p
            P = C.POINTER
            vp, i64, i32, dbl = C.c_void_p, C.c_int64, C.c_int32, C.c_double
            L.lcx_context_create.argtypes = [C.c_int, P(vp)]
            L.lcx_context_destroy.argtypes = [vp]
            L.lcx_set_profiling.argtypes = [vp, C.c_int]
            L.lcx_get_stats.argtypes = [vp, P(PrefillStatsC)]
            L.lcx_estimate_block.argtypes = [vp, P(AttentionInputC), i64, i64, i64, i64, i32,
                                             P(ChunkConfigC), vp, vp]
            L.lcx_line_scores.argtypes = [vp, P(AttentionInputC), i64, i64, i64, i64, i32,
                                          P(ChunkConfigC), i32, vp, vp, vp]
            L.lcx_select_from_scores.argtypes = [vp, vp, vp, i32, i64, i64, i64, i64,
                                                 P(SelectionOptionsC), vp, vp, i64, vp, vp,
                                                 i64, vp]
            L.lcx_select_critical.argtypes = [vp, vp, i32, i64, i64, i64, i64,
                                              P(SelectionOptionsC), vp, vp, i64, vp, vp, i64,
                                              vp]
            L.lcx_sparse_attention.argtypes = [vp, P(AttentionInputC), vp, vp, i64, vp, vp, i64,
                                               i32, P(ChunkConfigC), i32, vp, vp, vp]
            L.lcx_full_attention.argtypes = [vp, P(AttentionInputC), i32, P(ChunkConfigC), i32,
                                             vp, vp, vp]
            L.lcx_chunked_prefill.argtypes = [vp, P(AttentionInputC), P(PrefillConfigC),
                                              P(PrefillOutputC), vp]
            L.lcx_chunked_prefill_host.argtypes = [vp, P(AttentionInputC), P(PrefillConfigC),
                                                   P(PrefillOutputC), vp]
            L.lcx_attention_recall.argtypes = [vp, vp, vp, i64, dbl, vp, P(dbl), vp]
            L.lcx_lse_merge.argtypes = [vp, vp, vp, i32, i64, i32, vp, vp, vp]
            L.lcx_stream_wait_chunk.argtypes = [vp, i64, vp]
            L.lcx_get_chunk_ms.argtypes = [vp, vp, i64, P(i64)]
            L.lcx_lse_scale_partial.argtypes = [vp, vp, vp, vp, i32, i64, i32, i32, vp, vp]
            L.lcx_attention_rel.argtypes = [vp, P(AttentionInputC), vp, vp, i64, vp, vp, i64, vp,
                                            vp, vp, vp]
            _lib = L
    return _lib


def check(status: int) -> None:
    if status != 0:
        msg = lib().lcx_last_error().decode(errors="replace")
        raise Error(KINDS.get(status, f"status{status}"), msg)


class Context:
    """Owns an lcx_context (workspace, RoPE table) on one device."""

    def __init__(self, device: int = 0):
        self.ptr = C.c_void_p()
        check(lib().lcx_context_create(device, C.byref(self.ptr)))
        self.device = device

    def close(self):
        if self.ptr:
            lib().lcx_context_destroy(self.ptr)
            self.ptr = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def stats(self) -> dict:
        s = PrefillStatsC()
        check(lib().lcx_get_stats(self.ptr, C.byref(s)))
        return {f: getattr(s, f) for f, _ in PrefillStatsC._fields_}

    def chunk_ms(self) -> list:
        """Per-chunk device ms of the last chunked prefill (profiling on)."""
        cnt = C.c_int64(0)
        check(lib().lcx_get_chunk_ms(self.ptr, None, 0, C.byref(cnt)))
        buf = (C.c_float * max(1, cnt.value))()
        check(lib().lcx_get_chunk_ms(self.ptr, buf, cnt.value, C.byref(cnt)))
        return [float(buf[i]) for i in range(cnt.value)]

    def set_profiling(self, on: bool):
        check(lib().lcx_set_profiling(self.ptr, int(on)))


_contexts: dict[int, Context] = {}


def context(device: int | None = None) -> Context:
    import torch
    if device is None:
        device = torch.cuda.current_device()
    if device not in _contexts:
        _contexts[device] = Context(device)
    return _contexts[device]
