"""Python mirror of the reference ``longctx`` operator API for the prefill path.

Same names, argument meaning and error kinds as the C++ reference
(/root/reference/proj/core/include/longctx/{attention,dca,sparse,refine}.hpp), so
code written against the reference reads the same here.  Matrices are numpy
arrays (n x D) like ``longctx::Matrix``; every operator uploads to the GPU, runs the
sm_100a kernels through the C-ABI (include/longctx_b200.h) and returns host
results.  ``precision`` selects the device storage type of q/k/v: "fp32" (the
parity path, exact fp32 math) or "bf16".

There is no CPU fallback: without the built library and an sm_100 device every
operator raises ``Error(kind="cuda")``.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from enum import Enum

import numpy as np

from . import device as dev
from ._lib import Error

DEFAULT_ROPE_BASE = 10000.0   # attention.hpp:11


class PositionMode(Enum):     # sparse.hpp:63
    Standard = 0
    DcaContinuous = 1


class PrefillMode(Enum):      # sparse.hpp:97
    Full = 0
    Sparse = 1


@dataclass(frozen=True)
class HeadBudget:             # sparse.hpp:17-23
    vertical: int = 0
    slash: int = 0

    def total(self) -> int:
        return self.vertical + self.slash


@dataclass(frozen=True)
class SelectionOptions:       # sparse.hpp:65-69
    force_sink_column: bool = True
    force_local_band: bool = True
    slash_mean: bool = True

    def dev(self) -> dev.Options:
        return dev.Options(self.force_sink_column, self.force_local_band, self.slash_mean)


@dataclass(frozen=True)
class ChunkConfig:            # dca.hpp:15-25
    chunk_size: int = 0
    train_len: int = 0
    local_window: int = 0

    @staticmethod
    def with_default_window(chunk_size: int, train_len: int) -> "ChunkConfig":
        w = min(chunk_size, train_len - chunk_size if train_len > chunk_size else 0)
        cfg = ChunkConfig(chunk_size, train_len, w)
        cfg.validate()
        return cfg

    def validate(self):       # dca.cpp:18-30
        if self.chunk_size == 0:
            raise Error("config", "chunkSize must be positive")
        if self.train_len == 0:
            raise Error("config", "trainLen must be positive")
        if self.chunk_size > self.train_len:
            raise Error("config", "chunkSize must not exceed trainLen")
        if self.local_window > min(self.chunk_size, self.train_len - self.chunk_size):
            raise Error("config",
                        "localWindow must not exceed min(chunkSize, trainLen - chunkSize)")

    def tuple(self):
        return (self.chunk_size, self.train_len, self.local_window)


def yarn_temperature(scale_factor: float) -> float:   # dca.cpp:32-37
    if not scale_factor > 0.0:
        raise Error("domain", "scale factor must be positive")
    if scale_factor <= 1.0:
        return 1.0
    root = 0.1 * math.log(scale_factor) + 1.0
    return 1.0 / (root * root)


@dataclass(frozen=True)
class YarnScale:              # dca.hpp:31-37
    scale_factor: float = 1.0
    temperature: float = 1.0

    @staticmethod
    def from_scale(s: float) -> "YarnScale":
        return YarnScale(s, yarn_temperature(s))


def dca_relative(i: int, j: int, cfg: ChunkConfig) -> int:   # dca.cpp:62-80
    if j > i:
        raise Error("causality", "classify_pair requires j <= i")
    s, c = cfg.chunk_size, cfg.train_len
    qc, kc = i // s, j // s
    if qc == kc:
        qpos = i % s
    elif qc == kc + 1:
        qpos = min(i % s + s, c - 1)
    else:
        qpos = c - 1
    return qpos - j % s


def selection_position(i: int, j: int, cfg: ChunkConfig) -> int:   # sparse.cpp:137-140
    if j > i:
        raise Error("causality", "selection_position requires j <= i")
    return min(i - j, cfg.train_len - 1)


@dataclass
class AttentionInput:         # attention.hpp:15-30
    q: np.ndarray
    k: np.ndarray
    v: np.ndarray
    positions_q: np.ndarray | None = None
    positions_k: np.ndarray | None = None
    rope_base: float = DEFAULT_ROPE_BASE
    temperature: float = 1.0

    def seq_len(self) -> int:
        return int(np.asarray(self.q).shape[0])

    def head_dim(self) -> int:
        return int(np.asarray(self.q).shape[1])

    def validate(self):       # attention.cpp:70-94
        q, k, v = (np.asarray(x) for x in (self.q, self.k, self.v))
        n, d = q.shape
        if k.shape != (n, d) or v.shape != (n, d):
            raise Error("dimension", "attention input matrices must share n and D")
        if n == 0:
            raise Error("dimension", "attention input must have at least one row")
        if d == 0 or d % 2:
            raise Error("config", "head dimension must be even and positive (rope pairs)")
        pq = np.arange(n) if self.positions_q is None else np.asarray(self.positions_q)
        pk = np.arange(n) if self.positions_k is None else np.asarray(self.positions_k)
        if len(pq) != n or len(pk) != n:
            raise Error("dimension", "positions length must equal row count")
        if (pq < 0).any():
            raise Error("domain", "query positions must be non-negative")
        if (pk < 0).any():
            raise Error("domain", "key positions must be non-negative")
        if not self.rope_base > 0.0:
            raise Error("domain", "rope base must be positive")
        if not self.temperature > 0.0:
            raise Error("domain", "temperature must be positive")
        if not (np.isfinite(q).all() and np.isfinite(k).all() and np.isfinite(v).all()):
            raise Error("domain", "attention input values must be finite")


@dataclass
class AttentionResult:        # attention.hpp:32-35
    output: np.ndarray
    lse: np.ndarray


@dataclass
class CriticalSet:            # sparse.hpp:40-58
    verticals: list = field(default_factory=list)
    slashes: list = field(default_factory=list)
    context_length: int = 0

    def admits(self, i: int, j: int) -> bool:
        if j in set(self.verticals):
            return True
        return j <= i and (i - j) in set(self.slashes)

    def admitted_row(self, i: int) -> list:
        vs = [v for v in self.verticals if v <= i]
        ss = [i - d for d in self.slashes if d <= i]
        row = sorted(set(vs) | set(ss))
        return row if row else [i]

    def admitted_count(self) -> int:
        return sum(len(self.admitted_row(i)) for i in range(self.context_length))

    def to_json(self) -> dict:
        return {"contextLength": self.context_length, "verticals": list(self.verticals),
                "slashes": list(self.slashes)}

    @staticmethod
    def from_json(j: dict) -> "CriticalSet":
        return CriticalSet(sorted(set(j["verticals"])), sorted(set(j["slashes"])),
                           int(j["contextLength"]))


def density(crit: CriticalSet) -> float:   # sparse.cpp:286-291
    n = crit.context_length
    if n == 0:
        raise Error("dimension", "critical set has no context")
    return crit.admitted_count() / (n * (n + 1) / 2.0)


@dataclass
class ChunkSelection:         # sparse.hpp:99-104
    chunk_index: int
    begin: int
    end: int
    critical: CriticalSet


@dataclass
class PrefillState:           # sparse.hpp:107-113
    cached_k: np.ndarray
    cached_v: np.ndarray
    selections: list
    chunk_len: int
    last_q: int


@dataclass
class PrefillResult:
    result: AttentionResult
    state: PrefillState


# ---------------------------------------------------------------- helpers --
def _torch():
    import torch
    if not torch.cuda.is_available():
        raise Error("cuda", "no CUDA device: the sm_100a path has no CPU fallback")
    return torch


def _to_dev(x, precision):
    torch = _torch()
    t = torch.as_tensor(np.ascontiguousarray(x, dtype=np.float64))
    t = t.to(torch.float32 if precision == "fp32" else torch.bfloat16)
    return t.cuda()


def _heads(mat, precision):
    """n x D host matrix -> [n, 1, D] device tensor."""
    return _to_dev(mat, precision).unsqueeze(1).contiguous()


def _pos(p, n):
    if p is None:
        return None
    torch = _torch()
    return torch.as_tensor(np.asarray(p, dtype=np.int64)).cuda()


def _lists_to_dev(crit: CriticalSet):
    torch = _torch()
    v = torch.tensor([list(crit.verticals) or [0]], dtype=torch.int32).cuda()
    s = torch.tensor([list(crit.slashes) or [0]], dtype=torch.int32).cuda()
    nv = torch.tensor([len(crit.verticals)], dtype=torch.int32).cuda()
    ns = torch.tensor([len(crit.slashes)], dtype=torch.int32).cuda()
    return v, nv, s, ns


def _result(out, lse):
    return AttentionResult(out[:, 0, :].double().cpu().numpy(), lse[0].double().cpu().numpy())


# -------------------------------------------------------------- operators --
def estimate_block(q, k, last_q: int, mode: PositionMode, cfg: ChunkConfig | None,
                   rope_base: float = DEFAULT_ROPE_BASE, precision: str = "fp32") -> np.ndarray:
    """sparse.hpp:74-76 -- probabilities of the trailing min(last_q, q.rows) rows."""
    q, k = np.asarray(q), np.asarray(k)
    if last_q == 0:
        raise Error("config", "lastQ must be positive")
    if q.shape[1] != k.shape[1]:
        raise Error("dimension", "query/key dimensions differ")
    if q.shape[1] == 0 or q.shape[1] % 2:
        raise Error("config", "head dimension must be even")
    if q.shape[0] == 0 or k.shape[0] == 0:
        raise Error("dimension", "empty query or key matrix")
    if q.shape[0] > k.shape[0]:
        raise Error("dimension", "queries must be the trailing rows of the key timeline")
    if mode == PositionMode.DcaContinuous and cfg is None:
        raise Error("config", "dcaContinuous estimation requires a chunk config")
    nq, nk, d = q.shape[0], k.shape[0], q.shape[1]
    qfull = np.zeros((nk, d))
    qfull[nk - nq:] = q
    est = dev.estimate_block(_heads(qfull, precision), _heads(k, precision), q_row0=nk - nq,
                             nq=nq, nk=nk, last_q=last_q,
                             position_mode="dca_continuous" if mode == PositionMode.DcaContinuous
                             else "standard", dca=cfg.tuple() if cfg else None,
                             rope_base=rope_base)
    return est[0].double().cpu().numpy()


def select_critical(est, budget: HeadBudget, n: int,
                    opts: SelectionOptions = SelectionOptions()) -> CriticalSet:
    """sparse.hpp:81-82 (scores reduced in fp32 on the device)."""
    torch = _torch()
    est = np.asarray(est)
    if est.shape[1] != n:
        raise Error("dimension", "estimation block must have n columns")
    if est.shape[0] == 0 or est.shape[0] > n:
        raise Error("dimension", "estimation block row count out of range")
    e = torch.as_tensor(est, dtype=torch.float32).cuda().unsqueeze(0).contiguous()
    v, nv, s, ns = dev.select_critical(e, n=n, budget=(budget.vertical, budget.slash),
                                       opts=opts.dev())
    return CriticalSet(v[0, :int(nv[0])].tolist(), s[0, :int(ns[0])].tolist(), n)


def sparse_attention(inp: AttentionInput, crit: CriticalSet,
                     rel_override: ChunkConfig | None = None,
                     precision: str = "fp32") -> AttentionResult:
    """sparse.hpp:87-88.  rel_override: the reference passes the RelPositionMatrix built by
    dca_position_matrix(n, cfg); here the ChunkConfig itself (the kernel remaps in-flight)."""
    inp.validate()
    n = inp.seq_len()
    if crit.context_length != n:
        raise Error("dimension", "critical set context length must equal n")
    if rel_override is not None:
        rel_override.validate()
    v, nv, s, ns = _lists_to_dev(crit)
    out, lse = dev.sparse_attention(
        _heads(inp.q, precision), _heads(inp.k, precision), _heads(inp.v, precision), v, nv, s,
        ns, dca=rel_override.tuple() if rel_override else None,
        positions_q=None if rel_override else _pos(inp.positions_q, n),
        positions_k=None if rel_override else _pos(inp.positions_k, n),
        rope_base=inp.rope_base, temperature=inp.temperature)
    return _result(out, lse)


def full_attention(inp: AttentionInput, rel_override: ChunkConfig | None = None,
                   precision: str = "fp32") -> AttentionResult:
    """attention.hpp:57-58."""
    inp.validate()
    n = inp.seq_len()
    if rel_override is not None:
        rel_override.validate()
    out, lse = dev.full_attention(
        _heads(inp.q, precision), _heads(inp.k, precision), _heads(inp.v, precision),
        dca=rel_override.tuple() if rel_override else None,
        positions_q=None if rel_override else _pos(inp.positions_q, n),
        positions_k=None if rel_override else _pos(inp.positions_k, n),
        rope_base=inp.rope_base, temperature=inp.temperature)
    return _result(out, lse)


def dca_attention(inp: AttentionInput, cfg: ChunkConfig, yarn: YarnScale,
                  precision: str = "fp32") -> AttentionResult:
    """dca.hpp:64-65 / dca.cpp:93-113."""
    cfg.validate()
    if not yarn.scale_factor > 0.0:
        raise Error("domain", "scale factor must be positive")
    if yarn.temperature != yarn_temperature(yarn.scale_factor):
        raise Error("config", "temperature inconsistent with scale factor")
    n = inp.seq_len()
    eff = AttentionInput(inp.q, inp.k, inp.v, np.arange(n), np.arange(n), inp.rope_base,
                         yarn.temperature)
    if n <= cfg.chunk_size and yarn.scale_factor <= 1.0:
        return full_attention(eff, None, precision)
    return full_attention(eff, cfg, precision)


def chunked_prefill(inp: AttentionInput, chunk_len: int, last_q: int, budget: HeadBudget,
                    mode: PrefillMode, pos_mode: PositionMode, cfg: ChunkConfig | None,
                    opts: SelectionOptions = SelectionOptions(),
                    precision: str = "fp32") -> PrefillResult:
    """sparse.hpp:125-129."""
    inp.validate()
    if chunk_len == 0:
        raise Error("config", "chunkLen must be positive")
    if last_q == 0:
        raise Error("config", "lastQ must be positive")
    if mode == PrefillMode.Sparse and chunk_len < last_q:
        raise Error("config", "sparse prefill requires chunkLen >= lastQ")
    if pos_mode == PositionMode.DcaContinuous:
        if cfg is None:
            raise Error("config", "dcaContinuous prefill requires a chunk config")
        cfg.validate()
    n = inp.seq_len()
    dca = pos_mode == PositionMode.DcaContinuous
    r = dev.chunked_prefill(
        _heads(inp.q, precision), _heads(inp.k, precision), _heads(inp.v, precision),
        chunk_len=chunk_len, last_q=last_q, budget=(budget.vertical, budget.slash),
        mode="sparse" if mode == PrefillMode.Sparse else "full",
        position_mode="dca_continuous" if dca else "standard",
        dca=cfg.tuple() if dca else None, opts=opts.dev(),
        positions_q=_pos(inp.positions_q, n), positions_k=_pos(inp.positions_k, n),
        rope_base=inp.rope_base, temperature=inp.temperature)
    sels = []
    if mode == PrefillMode.Sparse:
        V, NV, S, NS = (r[x].cpu() for x in ("verticals", "nv", "slashes", "ns"))
        for ci in range(V.shape[0]):
            t0, t1 = ci * chunk_len, min(n, (ci + 1) * chunk_len)
            sels.append(ChunkSelection(ci, t0, t1, CriticalSet(
                V[ci, 0, :int(NV[ci, 0])].tolist(), S[ci, 0, :int(NS[ci, 0])].tolist(), t1)))
    res = _result(r["out"], r["lse"])
    st = PrefillState(np.asarray(inp.k), np.asarray(inp.v), sels, chunk_len, last_q)
    return PrefillResult(res, st)


@dataclass
class RecallReport:           # refine.hpp:15-20
    layer: int = 0
    head: int = 0
    per_query: np.ndarray = None
    aggregate: float = 0.0


def attention_recall(lse_sparse, lse_full, slack: float = 1e-5) -> RecallReport:
    """refine.hpp:25-26 (slack scaled to fp32; the reference's 1e-12 is fp64-only)."""
    torch = _torch()
    a = np.asarray(lse_sparse, dtype=np.float64)
    b = np.asarray(lse_full, dtype=np.float64)
    if a.shape != b.shape:
        raise Error("dimension", "recall needs equally many sparse and full lse values")
    if a.size == 0:
        raise Error("dimension", "recall needs at least one query")
    per, agg = dev.attention_recall(torch.as_tensor(a, dtype=torch.float32).cuda(),
                                    torch.as_tensor(b, dtype=torch.float32).cuda(), slack=slack)
    return RecallReport(per_query=per.double().cpu().numpy(), aggregate=agg)


@dataclass
class RecallMeasurement:      # refine.hpp:28-34
    last_q: int = 64
    selection: SelectionOptions = SelectionOptions()
    aggregate: str = "mean"   # or "fraction_above"
    fraction_tau: float = 0.9


def measure_budget_recall(inp: AttentionInput, budget: HeadBudget,
                          measure: RecallMeasurement = RecallMeasurement(),
                          precision: str = "fp32") -> float:
    """refine.cpp:74-85: full vs sparse (Standard positions, all rows, one shot)."""
    n = inp.seq_len()
    full = full_attention(inp, None, precision)
    est = estimate_block(inp.q, inp.k, min(measure.last_q, n), PositionMode.Standard, None,
                         inp.rope_base, precision)
    crit = select_critical(est, budget, n, measure.selection)
    sp = sparse_attention(inp, crit, None, precision)
    rep = attention_recall(sp.lse, full.lse, slack=1e-5 if precision == "fp32" else 4e-3)
    if measure.aggregate == "mean":
        return float(np.mean(rep.per_query))
    return float(np.mean(rep.per_query >= measure.fraction_tau))
