"""ctypes front-end for the CPU oracle (TEST INFRASTRUCTURE ONLY).

Two back-ends with the same Python surface:
  * ``Oracle("port")``      -> oracle/build/liblongctx_oracle.so, the C restatement
                               (oracle/longctx_oracle.c) of the reference path;
  * ``Oracle("reference")`` -> oracle/_ref/liblongctx_ref.so, the reference library
                               itself compiled from /root/reference (oracle/Makefile).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this module, and only as the checker / CPU baseline.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_LIB = os.path.join(HERE, "build", "liblongctx_oracle.so")
REF_LIB = os.path.join(HERE, "_ref", "liblongctx_ref.so")

KINDS = {1: "dimension", 2: "config", 3: "domain", 4: "causality", 5: "empty_row",
         6: "empty_calibration"}


class OracleError(Exception):
    def __init__(self, code: int, msg: str = ""):
        self.code = code
        self.kind = KINDS.get(code, f"code{code}")
        super().__init__(f"{self.kind}: {msg}")


def _d(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _pd(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _pi(a):
    return a.ctypes.data_as(C.POINTER(C.c_int64))


def build() -> None:
    import subprocess
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def ref_available() -> bool:
    return os.path.exists(REF_LIB)


@dataclass
class Critical:
    verticals: list
    slashes: list
    context_length: int


@dataclass
class ChunkSel:
    chunk_index: int
    begin: int
    end: int
    critical: Critical


class Oracle:
    """Same call surface for the port and the compiled reference."""

    def __init__(self, kind: str = "port"):
        self.kind = kind
        path = PORT_LIB if kind == "port" else REF_LIB
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        self.lib = C.CDLL(path)
        self.p = "lco_" if kind == "port" else "ref_"
        if kind == "reference":
            self.lib.ref_last_error.restype = C.c_char_p
            self.lib.ref_yarn_temperature.restype = C.c_double
            self.lib.ref_yarn_temperature.argtypes = [C.c_double]
            self.lib.ref_module_seed.restype = C.c_uint64
            self.lib.ref_module_seed.argtypes = [C.c_uint64, C.c_char_p]
            self.lib.ref_dca_relative.restype = C.c_int64
            self.lib.ref_dca_relative.argtypes = [C.c_int64] * 5
        else:
            self.lib.lco_yarn_temperature.restype = C.c_double
            self.lib.lco_yarn_temperature.argtypes = [C.c_double]
            self.lib.lco_dca_relative.restype = C.c_int64
            self.lib.lco_dca_relative.argtypes = [C.c_int64] * 4
            self.lib.lco_admitted_count.restype = C.c_int64

    def _check(self, st):
        if st:
            msg = self.lib.ref_last_error().decode() if self.kind == "reference" else ""
            raise OracleError(st, msg)

    # -- scalars ------------------------------------------------------------
    def yarn_temperature(self, s: float) -> float:
        return getattr(self.lib, self.p + "yarn_temperature")(s)

    def dca_relative(self, i, j, s, c, w=0):
        if self.kind == "reference":
            return self.lib.ref_dca_relative(i, j, s, c, w)
        return self.lib.lco_dca_relative(i, j, s, c)

    # -- estimator / selection ---------------------------------------------
    def estimate_block(self, q, k, last_q, pos_mode=0, cfg=None, rope_base=1e4):
        q, k = _d(q), _d(k)
        nq, dim = q.shape
        nk = k.shape[0]
        block = min(last_q, nq)
        est = np.zeros((max(block, 1), nk), np.float64)
        s, c, w = cfg if cfg else (0, 0, 0)
        if self.kind == "reference":
            st = self.lib.ref_estimate_block(_pd(q), C.c_int64(nq), _pd(k), C.c_int64(nk),
                                             C.c_int64(dim), C.c_int64(last_q), C.c_int(pos_mode),
                                             C.c_int64(s), C.c_int64(c), C.c_int64(w),
                                             C.c_double(rope_base), _pd(est))
        else:
            if pos_mode == 1 and cfg is None:
                raise OracleError(2, "dcaContinuous estimation requires a chunk config")
            st = self.lib.lco_estimate_block(_pd(q), C.c_int64(nq), _pd(k), C.c_int64(nk),
                                             C.c_int64(dim), C.c_int64(last_q), C.c_int(pos_mode),
                                             C.c_int64(c), C.c_double(rope_base), _pd(est))
        self._check(st)
        return est

    def select_critical(self, est, budget, n, force_sink=True, force_band=True, slash_mean=True):
        est = _d(est)
        rows = est.shape[0]
        bv, bs = budget
        cap_v, cap_s = bv + 2, bs + rows + 1
        ov, os_ = np.zeros(cap_v, np.int64), np.zeros(cap_s, np.int64)
        nv, ns = C.c_int64(), C.c_int64()
        if self.kind == "reference":
            st = self.lib.ref_select_critical(_pd(est), C.c_int64(rows), C.c_int64(n),
                                              C.c_int64(bv), C.c_int64(bs), C.c_int(force_sink),
                                              C.c_int(force_band), C.c_int(slash_mean), _pi(ov),
                                              C.c_int64(cap_v), C.byref(nv), _pi(os_),
                                              C.c_int64(cap_s), C.byref(ns))
        else:
            st = self.lib.lco_select_critical(_pd(est), C.c_int64(rows), C.c_int64(n),
                                              C.c_int64(bv), C.c_int64(bs), C.c_int(force_sink),
                                              C.c_int(force_band), C.c_int(slash_mean), _pi(ov),
                                              C.byref(nv), _pi(os_), C.byref(ns), None, None)
        self._check(st)
        return Critical(list(ov[:nv.value]), list(os_[:ns.value]), n)

    def select_from_scores(self, col, slash, n, block, budget, force_sink=True, force_band=True):
        """Port only: selection stage from already-reduced line scores."""
        col, slash = _d(col), _d(slash)
        bv, bs = budget
        ov, os_ = np.zeros(bv + 2, np.int64), np.zeros(bs + block + 1, np.int64)
        nv, ns = C.c_int64(), C.c_int64()
        self._check(self.lib.lco_select_from_scores(_pd(col), _pd(slash), C.c_int64(n),
                                                    C.c_int64(block), C.c_int64(bv),
                                                    C.c_int64(bs), C.c_int(force_sink),
                                                    C.c_int(force_band), _pi(ov), C.byref(nv),
                                                    _pi(os_), C.byref(ns)))
        return Critical(list(ov[:nv.value]), list(os_[:ns.value]), n)

    def line_scores(self, est, n, slash_mean=True):
        """Port only: (col_score, slash_score) exactly as select_critical forms them."""
        est = _d(est)
        rows = est.shape[0]
        col, sl = np.zeros(n), np.zeros(n)
        ov, os_ = np.zeros(2, np.int64), np.zeros(rows + 1, np.int64)
        nv, ns = C.c_int64(), C.c_int64()
        self._check(self.lib.lco_select_critical(_pd(est), C.c_int64(rows), C.c_int64(n),
                                                 C.c_int64(0), C.c_int64(0), C.c_int(0),
                                                 C.c_int(0), C.c_int(slash_mean), _pi(ov),
                                                 C.byref(nv), _pi(os_), C.byref(ns), _pd(col),
                                                 _pd(sl)))
        return col, sl

    def admitted_count(self, verticals, slashes, n):
        v, s = _i(verticals), _i(slashes)
        if self.kind == "reference":
            cnt, dens = C.c_int64(), C.c_double()
            self._check(self.lib.ref_admitted_count(_pi(v), C.c_int64(len(v)), _pi(s),
                                                    C.c_int64(len(s)), C.c_int64(n),
                                                    C.byref(cnt), C.byref(dens)))
            return cnt.value
        return self.lib.lco_admitted_count(_pi(v), C.c_int64(len(v)), _pi(s),
                                           C.c_int64(len(s)), C.c_int64(n))

    def density(self, verticals, slashes, n):
        return self.admitted_count(verticals, slashes, n) / (n * (n + 1) / 2.0)

    # -- attention ----------------------------------------------------------
    def _pos(self, n, pos):
        return _i(np.arange(n) if pos is None else pos)

    def sparse_attention(self, q, k, v, crit: Critical, pos_q=None, pos_k=None, rope_base=1e4,
                         temperature=1.0, dca=None):
        q, k, v = _d(q), _d(k), _d(v)
        n, dim = q.shape
        pq, pk = self._pos(n, pos_q), self._pos(n, pos_k)
        vv, ss = _i(crit.verticals), _i(crit.slashes)
        out, lse = np.zeros((n, dim)), np.zeros(n)
        s, c, w = dca if dca else (0, 0, 0)
        if self.kind == "reference":
            st = self.lib.ref_sparse_attention(_pd(q), _pd(k), _pd(v), C.c_int64(n),
                                               C.c_int64(dim), _pi(pq), _pi(pk),
                                               C.c_double(rope_base), C.c_double(temperature),
                                               _pi(vv), C.c_int64(len(vv)), _pi(ss),
                                               C.c_int64(len(ss)), C.c_int(dca is not None),
                                               C.c_int64(s), C.c_int64(c), C.c_int64(w),
                                               _pd(out), _pd(lse))
        else:
            st = self.lib.lco_sparse_attention(_pd(q), _pd(k), _pd(v), C.c_int64(n),
                                               C.c_int64(dim), _pi(pq), _pi(pk),
                                               C.c_double(rope_base), C.c_double(temperature),
                                               _pi(vv), C.c_int64(len(vv)), _pi(ss),
                                               C.c_int64(len(ss)), C.c_int(dca is not None),
                                               C.c_int64(s), C.c_int64(c), _pd(out), _pd(lse))
        self._check(st)
        return out, lse

    def full_attention(self, q, k, v, pos_q=None, pos_k=None, rope_base=1e4, temperature=1.0,
                       dca=None):
        q, k, v = _d(q), _d(k), _d(v)
        n, dim = q.shape
        pq, pk = self._pos(n, pos_q), self._pos(n, pos_k)
        out, lse = np.zeros((n, dim)), np.zeros(n)
        s, c, w = dca if dca else (0, 0, 0)
        if self.kind == "reference":
            st = self.lib.ref_full_attention(_pd(q), _pd(k), _pd(v), C.c_int64(n), C.c_int64(dim),
                                             _pi(pq), _pi(pk), C.c_double(rope_base),
                                             C.c_double(temperature), C.c_int(dca is not None),
                                             C.c_int64(s), C.c_int64(c), C.c_int64(w), _pd(out),
                                             _pd(lse))
        else:
            st = self.lib.lco_full_attention(_pd(q), _pd(k), _pd(v), C.c_int64(n), C.c_int64(dim),
                                             _pi(pq), _pi(pk), C.c_double(rope_base),
                                             C.c_double(temperature), C.c_int(dca is not None),
                                             C.c_int64(s), C.c_int64(c), _pd(out), _pd(lse))
        self._check(st)
        return out, lse

    def attention_rows(self, q, k, v, rows, crit: Critical | None = None, pos_q=None,
                       pos_k=None, rope_base=1e4, temperature=1.0, dca=None):
        """Port only: sparse (crit) or dense (crit None) attention of the listed rows."""
        q, k, v = _d(q), _d(k), _d(v)
        n, dim = q.shape
        pq, pk = self._pos(n, pos_q), self._pos(n, pos_k)
        rows = _i(rows)
        vv = _i(crit.verticals if crit else [0])
        ss = _i(crit.slashes if crit else [0])
        out, lse = np.zeros((len(rows), dim)), np.zeros(len(rows))
        s, c, w = dca if dca else (0, 0, 0)
        fn = self.lib.lco_attention_row_list
        self._check(fn(_pd(q), _pd(k), _pd(v), C.c_int64(n), C.c_int64(dim), _pi(pq), _pi(pk),
                       C.c_double(rope_base), C.c_double(temperature), _pi(vv),
                       C.c_int64(len(crit.verticals) if crit else 0), _pi(ss),
                       C.c_int64(len(crit.slashes) if crit else 0), C.c_int(crit is None),
                       C.c_int(dca is not None), C.c_int64(s), C.c_int64(c), _pi(rows),
                       C.c_int64(len(rows)), _pd(out), _pd(lse)))
        return out, lse

    def dca_attention(self, q, k, v, cfg, scale_factor, rope_base=1e4):
        q, k, v = _d(q), _d(k), _d(v)
        n, dim = q.shape
        s, c, w = cfg
        out, lse = np.zeros((n, dim)), np.zeros(n)
        fn = getattr(self.lib, self.p + "dca_attention")
        self._check(fn(_pd(q), _pd(k), _pd(v), C.c_int64(n), C.c_int64(dim),
                       C.c_double(rope_base), C.c_int64(s), C.c_int64(c), C.c_int64(w),
                       C.c_double(scale_factor), _pd(out), _pd(lse)))
        return out, lse

    def chunked_prefill(self, q, k, v, chunk_len, last_q, budget, mode="sparse",
                        pos_mode=0, cfg=None, force_sink=True, force_band=True, slash_mean=True,
                        pos_q=None, pos_k=None, rope_base=1e4, temperature=1.0):
        q, k, v = _d(q), _d(k), _d(v)
        n, dim = q.shape
        pq, pk = self._pos(n, pos_q), self._pos(n, pos_k)
        bv, bs = budget
        nch = max(1, -(-n // max(chunk_len, 1)))
        cap_v, cap_s = bv + 2, bs + last_q + 1
        sv, snv = np.zeros(nch * cap_v, np.int64), np.zeros(nch, np.int64)
        ss, sns = np.zeros(nch * cap_s, np.int64), np.zeros(nch, np.int64)
        out, lse = np.zeros((n, dim)), np.zeros(n)
        s, c, w = cfg if cfg else (0, 0, 0)
        m = 1 if mode == "sparse" else 0
        fn = getattr(self.lib, self.p + "chunked_prefill")
        if self.kind == "port" and pos_mode == 1 and cfg is None:
            raise OracleError(2, "dcaContinuous prefill requires a chunk config")
        st = fn(_pd(q), _pd(k), _pd(v), C.c_int64(n), C.c_int64(dim), _pi(pq), _pi(pk),
                C.c_double(rope_base), C.c_double(temperature), C.c_int64(chunk_len),
                C.c_int64(last_q), C.c_int64(bv), C.c_int64(bs), C.c_int(m), C.c_int(pos_mode),
                C.c_int64(s), C.c_int64(c), C.c_int64(w), C.c_int(force_sink),
                C.c_int(force_band), C.c_int(slash_mean), _pd(out), _pd(lse), _pi(sv), _pi(snv),
                C.c_int64(cap_v), _pi(ss), _pi(sns), C.c_int64(cap_s))
        self._check(st)
        sels = []
        if m == 1:
            for ci in range(nch):
                t0, t1 = ci * chunk_len, min(n, (ci + 1) * chunk_len)
                sels.append(ChunkSel(ci, t0, t1, Critical(
                    list(sv[ci * cap_v: ci * cap_v + snv[ci]]),
                    list(ss[ci * cap_s: ci * cap_s + sns[ci]]), t1)))
        return out, lse, sels

    # -- recall -------------------------------------------------------------
    def attention_recall(self, lse_sparse, lse_full, slack=1e-12):
        a, b = _d(lse_sparse), _d(lse_full)
        n = len(a)
        per = np.zeros(max(n, 1))
        agg = C.c_double()
        if self.kind == "reference":
            st = self.lib.ref_attention_recall(_pd(a), _pd(b), C.c_int64(n), _pd(per),
                                               C.byref(agg))
        else:
            st = self.lib.lco_attention_recall(_pd(a), _pd(b), C.c_int64(n), C.c_double(slack),
                                               _pd(per), C.byref(agg))
        self._check(st)
        return per[:n], agg.value

    # -- fixtures -----------------------------------------------------------
    def make_planted(self, n, dim, rope_base=1e4, vertical_columns=(), slash_offsets=(),
                     strength=10.0, vertical_strength=0.0, slash_strength=0.0, query_noise=1.0,
                     shared_scale=2.0, seed=0, dca=None, carrier_pairs=()):
        vc, so, cp = _i(list(vertical_columns) or [0]), _i(list(slash_offsets) or [0]), \
            _i(list(carrier_pairs) or [0])
        q, k, v = np.zeros((n, dim)), np.zeros((n, dim)), np.zeros((n, dim))
        s, c, w = dca if dca else (0, 0, 0)
        fn = getattr(self.lib, self.p + "make_planted")
        fn.argtypes = [C.c_int64, C.c_int64, C.c_double, C.POINTER(C.c_int64), C.c_int64,
                       C.POINTER(C.c_int64), C.c_int64, C.c_double, C.c_double, C.c_double,
                       C.c_double, C.c_double, C.c_uint64, C.c_int, C.c_int64, C.c_int64,
                       C.c_int64, C.POINTER(C.c_int64), C.c_int64, C.POINTER(C.c_double),
                       C.POINTER(C.c_double), C.POINTER(C.c_double)]
        self._check(fn(n, dim, rope_base, _pi(vc), len(vertical_columns), _pi(so),
                       len(slash_offsets), strength, vertical_strength, slash_strength,
                       query_noise, shared_scale, seed, int(dca is not None), s, c, w, _pi(cp),
                       len(carrier_pairs), _pd(q), _pd(k), _pd(v)))
        return q, k, v

    def random_input(self, seed, n, dim):
        """Port only: testutil::random_input (q, k, v uniform(-1,1), fresh mt19937_64(seed))."""
        q, k, v = np.zeros((n, dim)), np.zeros((n, dim)), np.zeros((n, dim))
        self.lib.lco_random_input(C.c_uint64(seed), C.c_int64(n), C.c_int64(dim), _pd(q), _pd(k),
                                  _pd(v))
        return q, k, v


class Rng:
    """Port-side std::mt19937_64 stream (to draw several random_inputs from one rng,
    as the reference tests do)."""

    def __init__(self, oracle: Oracle, seed: int):
        self.o = oracle
        self.buf = C.create_string_buffer(oracle.lib.lco_mt64_size())
        oracle.lib.lco_mt64_seed(self.buf, C.c_uint64(seed))

    def random_input(self, n, dim):
        q, k, v = np.zeros((n, dim)), np.zeros((n, dim)), np.zeros((n, dim))
        self.o.lib.lco_random_input_from(self.buf, C.c_int64(n), C.c_int64(dim), _pd(q), _pd(k),
                                         _pd(v))
        return q, k, v

    def next_u64(self):
        self.o.lib.lco_mt64_next.restype = C.c_uint64
        return self.o.lib.lco_mt64_next(self.buf)


# ---------------------------------------------------------------------------------------
# Fast fp64 restatement of the estimator's line scores for the large parity cases
# (t1 up to 1M keys, where the per-entry-RoPE loop of lco_estimate_block takes minutes per
# head).  Same math as sparse.cpp:142-188 (estimate_block) + 196-218 (line sums), using
# rope(q, gi - j) . k == rope(q, gi) . rope(k, j) (exact in real arithmetic; ~1e-15 apart
# in fp64, pinned against lco_estimate_block in tests/test_oracle_pin.py) and, for the
# DcaContinuous far region (gi - j > c - 1), rope(q, c - 1) . k_j.
def rope_rows(x, pos, rope_base):
    """x [m, dim] rotated by positions pos [m] (attention.cpp:14-33, fp64 angles)."""
    x = np.asarray(x, np.float64)
    dim = x.shape[1]
    th = np.power(float(rope_base), -np.arange(0, dim, 2, dtype=np.float64) / dim)
    ang = np.asarray(pos, np.float64)[:, None] * th[None, :]
    c, s = np.cos(ang), np.sin(ang)
    xe, xo = x[:, 0::2], x[:, 1::2]
    out = np.empty_like(x)
    out[:, 0::2] = xe * c - xo * s
    out[:, 1::2] = xe * s + xo * c
    return out


def estimate_probs_fast(q_rows, k, pos_mode=0, c=0, rope_base=1e4):
    """est [B, t1] of estimate_block for the chunk's last B query rows q_rows (global rows
    t1 - B .. t1 - 1) against keys k [t1, dim]."""
    q_rows, k = np.asarray(q_rows, np.float64), np.asarray(k, np.float64)
    B, dim = q_rows.shape
    t1 = k.shape[0]
    gi = np.arange(t1 - B, t1)
    j = np.arange(t1)
    logits = rope_rows(q_rows, gi, rope_base) @ rope_rows(k, j, rope_base).T
    if pos_mode == 1:
        far = (gi[:, None] - j[None, :]) > c - 1
        if far.any():
            lf = rope_rows(q_rows, np.full(B, c - 1), rope_base) @ k.T
            logits = np.where(far, lf, logits)
    logits /= np.sqrt(dim)
    logits[j[None, :] > gi[:, None]] = -np.inf
    logits -= logits.max(axis=1, keepdims=True)
    np.exp(logits, out=logits)
    logits /= logits.sum(axis=1, keepdims=True)
    return logits


def line_scores_fast(est, slash_mean=True):
    """(col_score, slash_score) of an est [B, t1] block exactly as select_critical forms
    them (sparse.cpp:196-218): column sums; per diagonal d = gi - j the sum (or mean over
    its entries), -inf for empty bins."""
    B, t1 = est.shape
    col = est.sum(axis=0)
    ssum = np.zeros(t1)
    for r in range(B):
        g = t1 - B + r
        ssum[:g + 1] += est[r, g::-1]
    d = np.arange(t1)
    cnt = np.minimum(B, t1 - d)
    score = ssum / cnt if slash_mean else ssum
    return col, score
