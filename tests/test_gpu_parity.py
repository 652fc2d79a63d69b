"""GPU parity: the sm_100a path (through the C-ABI) vs the CPU oracle on the same inputs.

Tolerances (D1): per row, max_d |o - o_ref| <= tol * max_d |o_ref| and
|lse - lse_ref| <= tol * max(|lse_ref|, 1), tol = 1e-5 (fp32 storage) / 2e-3 (bf16
storage); the oracle always receives exactly the values the device stores.
Index sets must be identical given identical fp32 scores (ties -> lowest index).
"""
import json
import os

import numpy as np
import pytest

from helpers import TOL, check_selection, lse_rel_err, rounded, row_rel_err

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def L():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2501_15383_b200 import longctx
    return longctx


@pytest.fixture(scope="module")
def D():
    from paper_2501_15383_b200 import device
    return device


def rin(port, seed, n, dim, precision):
    q, k, v = port.random_input(seed, n, dim)
    return rounded(q, precision), rounded(k, precision), rounded(v, precision)


# ----------------------------------------------------------------- estimator --
@pytest.mark.parametrize("precision", ["fp32", "bf16"])
@pytest.mark.parametrize("pm,cfg", [(0, None), (1, (32, 96, 32)), (1, (6, 10, 4))])
@pytest.mark.parametrize("n,dim,nq,lq", [(200, 16, 80, 64), (300, 128, 300, 64),
                                         (130, 8, 40, 100)])
def test_estimate_block(L, port, precision, pm, cfg, n, dim, nq, lq):
    q, k, _ = rin(port, n + dim, n, dim, precision)
    ref = port.estimate_block(q[n - nq:], k, lq, pm, cfg)
    mode = L.PositionMode.DcaContinuous if pm else L.PositionMode.Standard
    got = L.estimate_block(q[n - nq:], k, lq, mode, L.ChunkConfig(*cfg) if cfg else None,
                           precision=precision)
    assert got.shape == ref.shape
    # probabilities: row-relative (fp32 math on both storage types)
    assert row_rel_err(got, ref) <= 1e-5
    assert (got[ref == 0.0] == 0.0).all()  # causal zeros are exact


@pytest.mark.parametrize("pm,cfg", [(0, None), (1, (64, 192, 64))])
def test_line_scores_fused(D, port, pm, cfg):
    import torch
    n, dim, chunk, lq = 700, 128, 256, 64
    q, k, _ = rin(port, 5, n, dim, "fp32")
    est = port.estimate_block(q[n - chunk:], k, lq, pm, cfg)
    col_ref, sl_ref = port.line_scores(est, n)
    qt = torch.tensor(q, dtype=torch.float32).cuda().unsqueeze(1).contiguous()
    kt = torch.tensor(k, dtype=torch.float32).cuda().unsqueeze(1).contiguous()
    col, sl = D.line_scores(qt, kt, q_row0=n - chunk, nq=chunk, nk=n, last_q=lq,
                            position_mode="dca_continuous" if pm else "standard", dca=cfg)
    col, sl = col[0].double().cpu().numpy(), sl[0].double().cpu().numpy()
    assert np.abs(col - col_ref).max() <= 1e-5 * np.abs(col_ref).max()
    assert np.abs(sl - sl_ref).max() <= 1e-5 * np.abs(sl_ref).max()


@pytest.mark.parametrize("pm,cfg,n,nq", [(0, None, 2000, 512), (1, (256, 700, 256), 2000, 512),
                                         (1, (128, 384, 128), 1500, 64),
                                         (1, (64, 192, 64), 700, 256)])
@pytest.mark.parametrize("kind", ["normal", "peaked"])
def test_line_scores_tensor_core_bf16(D, port, pm, cfg, n, nq, kind):
    """The tcgen05 estimator (bf16 storage, head dim 128: 3-term bf16 split of the rotated
    operands, six products in fp32 TMEM) against the fp64 oracle on the same bf16 values,
    with far, mixed (CUDA-core) and near key tiles in one call."""
    import torch
    rng = np.random.default_rng(n + nq)
    q = rounded(rng.standard_normal((n, 1, 128)) * (1.7 if kind == "peaked" else 1.0), "bf16")
    k = rounded(rng.standard_normal((n, 1, 128)), "bf16")
    if kind == "peaked":
        k[rng.integers(0, n, n // 16)] *= 6.0
        k = rounded(k, "bf16")
    est = port.estimate_block(q[n - nq:, 0], k[:, 0], 64, pm, cfg)
    col_ref, sl_ref = port.line_scores(est, n)
    T = lambda x: torch.tensor(x).to(torch.bfloat16).cuda().contiguous()  # noqa: E731
    col, sl = D.line_scores(T(q), T(k), q_row0=n - nq, nq=nq, nk=n, last_q=64,
                            position_mode="dca_continuous" if pm else "standard", dca=cfg)
    col, sl = col[0].double().cpu().numpy(), sl[0].double().cpu().numpy()
    assert np.abs(col - col_ref).max() <= 1e-5 * np.abs(col_ref).max()
    assert np.abs(sl - sl_ref).max() <= 1e-5 * np.abs(sl_ref).max()


# ----------------------------------------------------------------- selection --
@pytest.mark.parametrize("seed", range(6))
def test_selection_identical_given_identical_scores(D, port, seed):
    """The GPU radix select vs the reference ranking (oracle select_from_scores) on the
    same fp32 scores, with heavy ties."""
    import torch
    rng = np.random.default_rng(seed)
    heads, n = 3, int(rng.integers(100, 5000))
    levels = int(rng.choice([3, 17, 1000, 1 << 20]))
    col = (rng.integers(0, levels, (heads, n)) / levels).astype(np.float32)
    sl = (rng.integers(0, levels, (heads, n)) / levels).astype(np.float32)
    block = int(rng.integers(1, min(64, n)))
    bud = (int(rng.integers(0, n // 2)), int(rng.integers(0, n // 2)))
    for sink, band in [(True, True), (False, False), (True, False)]:
        opts = D.Options(sink, band, True)
        v, nv, s, ns = D.select_from_scores(torch.tensor(col).cuda(), torch.tensor(sl).cuda(),
                                            block=block, budget=bud, opts=opts)
        for h in range(heads):
            exp = port.select_from_scores(col[h].astype(np.float64), sl[h].astype(np.float64), n,
                                          block, bud, sink, band)
            assert v[h, :int(nv[h])].tolist() == exp.verticals
            assert s[h, :int(ns[h])].tolist() == exp.slashes


@pytest.mark.parametrize("n,bud", [(4096, (100, 300)), (33333, (1000, 6096)),
                                   (262144, (1000, 6096)), (100000, (50000, 99990))])
def test_selection_cluster_path_large_n(D, port, n, bud):
    """The clustered radix select (8 CTAs per head, DSMEM histograms) on large score
    arrays with heavy ties and ties straddling the CTA slices: identical to the reference
    ranking (score desc, index asc) + forced lines."""
    import torch
    rng = np.random.default_rng(n)
    heads = 3
    col = rng.random((heads, n)).astype(np.float32)
    sl = rng.random((heads, n)).astype(np.float32)
    col[:, rng.integers(0, n, n // 3)] = 0.75  # a tie class spanning every slice
    sl[:, :] = np.round(sl * 64) / 64           # 65 tie classes
    block = 64
    T = lambda x: torch.tensor(x).cuda().contiguous()  # noqa: E731
    v, nv, s, ns = D.select_from_scores(T(col), T(sl), block=block, budget=bud)
    v, nv, s, ns = v.cpu().numpy(), nv.cpu().numpy(), s.cpu().numpy(), ns.cpu().numpy()
    for h in range(heads):
        exp = port.select_from_scores(col[h].astype(np.float64), sl[h].astype(np.float64), n,
                                      block, bud)
        assert v[h, :int(nv[h])].tolist() == exp.verticals
        assert s[h, :int(ns[h])].tolist() == exp.slashes


def test_select_critical_one_row_trick(L, ref):
    """Drive the REAL reference select_critical with a 1-row estimate (count 1 => mean =
    value) built from fp32 scores; the device selection must agree."""
    rng = np.random.default_rng(7)
    for n in [50, 777, 4096]:
        est = rng.random((1, n)).astype(np.float32).astype(np.float64)
        est[0, rng.integers(0, n, n // 3)] = 0.5  # ties
        for bud in [(3, 5), (n, 0), (0, n), (n // 2, n // 3)]:
            exp = ref.select_critical(est, bud, n)
            got = L.select_critical(est, L.HeadBudget(*bud), n)
            assert got.verticals == exp.verticals and got.slashes == exp.slashes


# ----------------------------------------------------------------- attention --
@pytest.mark.parametrize("precision", ["fp32", "bf16"])
@pytest.mark.parametrize("n", [512, 129, 1])
def test_sparse_attention_standard(L, port, precision, n):
    dim = 128
    q, k, v = rin(port, 11, n, dim, precision)
    crit = port.select_critical(port.estimate_block(q, k, 64), (20, 30), n)
    ref = port.sparse_attention(q, k, v, crit)
    got = L.sparse_attention(L.AttentionInput(q, k, v), L.CriticalSet(crit.verticals,
                                                                       crit.slashes, n),
                             precision=precision)
    assert row_rel_err(got.output, ref[0]) <= TOL[precision]
    assert lse_rel_err(got.lse, ref[1]) <= TOL[precision]


@pytest.mark.parametrize("cfg", [(64, 128, 64), (32, 80, 32), (6, 10, 4)])
def test_sparse_attention_dca_override(L, port, cfg):
    n, dim = 400, 32
    q, k, v = rin(port, 12, n, dim, "fp32")
    crit = port.select_critical(port.estimate_block(q, k, 32, 1, cfg), (10, 10), n)
    ref = port.sparse_attention(q, k, v, crit, dca=cfg, temperature=0.8)
    got = L.sparse_attention(L.AttentionInput(q, k, v, temperature=0.8),
                             L.CriticalSet(crit.verticals, crit.slashes, n), L.ChunkConfig(*cfg))
    assert row_rel_err(got.output, ref[0]) <= 1e-5
    assert lse_rel_err(got.lse, ref[1]) <= 1e-5


def test_sparse_attention_custom_positions(L, port):
    n, dim = 256, 16
    q, k, v = rin(port, 13, n, dim, "fp32")
    rng = np.random.default_rng(0)
    pq = np.sort(rng.integers(0, 5000, n))
    pk = np.sort(rng.integers(0, 5000, n))
    crit = port.select_critical(port.estimate_block(q, k, 16), (8, 8), n)
    ref = port.sparse_attention(q, k, v, crit, pos_q=pq, pos_k=pk, rope_base=500.0)
    got = L.sparse_attention(L.AttentionInput(q, k, v, pq, pk, rope_base=500.0),
                             L.CriticalSet(crit.verticals, crit.slashes, n))
    assert row_rel_err(got.output, ref[0]) <= 1e-5
    assert lse_rel_err(got.lse, ref[1]) <= 1e-5


@pytest.mark.parametrize("dca", [None, (48, 128, 48)])
@pytest.mark.parametrize("n", [300, 1])
def test_full_attention(L, port, dca, n):
    dim = 64
    q, k, v = rin(port, 14, n, dim, "fp32")
    ref = port.full_attention(q, k, v, dca=dca)
    got = L.full_attention(L.AttentionInput(q, k, v), L.ChunkConfig(*dca) if dca else None)
    assert row_rel_err(got.output, ref[0]) <= 1e-5
    assert lse_rel_err(got.lse, ref[1]) <= 1e-5


def test_dca_attention(L, port):
    n, dim = 260, 32
    q, k, v = rin(port, 15, n, dim, "fp32")
    for cfg, sf in [((64, 192, 64), 4.0), ((512, 1024, 256), 1.0)]:
        ref = port.dca_attention(q, k, v, cfg, sf)
        got = L.dca_attention(L.AttentionInput(q, k, v), L.ChunkConfig(*cfg),
                              L.YarnScale.from_scale(sf))
        assert row_rel_err(got.output, ref[0]) <= 1e-5
        assert lse_rel_err(got.lse, ref[1]) <= 1e-5


def test_full_coverage_equals_dense(L, port):
    """test_sparse.cpp:131-142."""
    n, dim = 64, 8
    q, k, v = rin(port, 5, n, dim, "fp32")
    inp = L.AttentionInput(q, k, v)
    sp = L.sparse_attention(inp, L.CriticalSet(list(range(n)), [], n))
    fu = L.full_attention(inp)
    assert np.abs(sp.output - fu.output).max() <= 1e-6
    assert np.abs(sp.lse - fu.lse).max() <= 1e-6


def test_self_diagonal_and_fallback_rows(L, port):
    """test_sparse.cpp:144-170."""
    q, k, v = rin(port, 6, 16, 8, "fp32")
    r = L.sparse_attention(L.AttentionInput(q, k, v), L.CriticalSet([], [0], 16))
    assert np.abs(r.output - v).max() <= 1e-6
    q, k, v = rin(port, 7, 8, 8, "fp32")
    r = L.sparse_attention(L.AttentionInput(q, k, v), L.CriticalSet([5], [], 8))
    assert np.abs(r.output[:5] - v[:5]).max() <= 1e-6
    r = L.sparse_attention(L.AttentionInput(q, k, v), L.CriticalSet([], [], 8))
    assert np.abs(r.output - v).max() <= 1e-6


# ------------------------------------------------------------ chunked prefill --
@pytest.mark.parametrize("name", ["sparsity_example.json", "sparsity_dca.json"])
@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_chunked_prefill_goldens(L, port, name, precision):
    """The reference's own example configs: identical per-chunk selections, recall and
    density reproduced, outputs within tolerance of the oracle on the same values."""
    from test_oracle_pin import planted_from_spec
    g = json.load(open(os.path.join(GOLD, name)))
    cfg, spec, exp = g["config"], g["spec"], g["expected"]
    q, k, v = (rounded(x, precision) for x in planted_from_spec(port, spec))
    dca = L.ChunkConfig(*cfg["chunk_cfg"]) if cfg["dca_mode"] else None
    pm = L.PositionMode.DcaContinuous if dca else L.PositionMode.Standard
    inp = L.AttentionInput(q, k, v, rope_base=spec["rope_base"])
    pr = L.chunked_prefill(inp, cfg["chunk_len"], cfg["last_q"], L.HeadBudget(*cfg["budget"]),
                           L.PrefillMode.Sparse, pm, dca, precision=precision)
    got_sel = [dict(verticals=s.critical.verticals, slashes=s.critical.slashes)
               for s in pr.state.selections]
    exp_sel = [dict(verticals=s["critical"]["verticals"], slashes=s["critical"]["slashes"])
               for s in exp["selections"]]
    assert got_sel == exp_sel
    out_ref, lse_ref, _ = port.chunked_prefill(q, k, v, cfg["chunk_len"], cfg["last_q"],
                                               tuple(cfg["budget"]), "sparse", 1 if dca else 0,
                                               dca.tuple() if dca else None,
                                               rope_base=spec["rope_base"])
    assert row_rel_err(pr.result.output, out_ref) <= TOL[precision]
    assert lse_rel_err(pr.result.lse, lse_ref) <= TOL[precision]
    # one-shot recall / density of the golden run, through the device path
    est = L.estimate_block(q, k, cfg["last_q"], pm, dca, spec["rope_base"], precision)
    crit = L.select_critical(est, L.HeadBudget(*cfg["budget"]), spec["n"])
    assert crit.verticals == exp["critical"]["verticals"]
    assert crit.slashes == exp["critical"]["slashes"]
    full = L.full_attention(inp, dca, precision)
    sp = L.sparse_attention(inp, crit, dca, precision)
    rec = L.attention_recall(sp.lse, full.lse, slack=1e-5 if precision == "fp32" else 4e-3)
    assert abs(rec.aggregate - exp["recall"]) <= (1e-6 if precision == "fp32" else 2e-3)
    assert L.density(crit) == exp["density"]


def test_chunked_prefill_kat_cases(L, port):
    g = json.load(open(os.path.join(GOLD, "kat_hashes.json")))
    for c in g["cases"]:
        q, k, v = port.random_input(c["seed"], c["n"], c["dim"])
        q, k, v = (rounded(x, "fp32") for x in (q, k, v))
        cfg = L.ChunkConfig(*c["cfg"]) if c["cfg"] else None
        pm = L.PositionMode.DcaContinuous if c["pos_mode"] else L.PositionMode.Standard
        pr = L.chunked_prefill(L.AttentionInput(q, k, v), c["chunk_len"], c["last_q"],
                               L.HeadBudget(*c["budget"]), L.PrefillMode.Sparse, pm, cfg)
        out_ref, lse_ref, sels = port.chunked_prefill(q, k, v, c["chunk_len"], c["last_q"],
                                                      tuple(c["budget"]), "sparse", c["pos_mode"],
                                                      c["cfg"] and tuple(c["cfg"]))
        for a, b in zip(pr.state.selections, sels):
            assert a.critical.verticals == b.critical.verticals
            assert a.critical.slashes == b.critical.slashes
        assert row_rel_err(pr.result.output, out_ref) <= 1e-5
        assert lse_rel_err(pr.result.lse, lse_ref) <= 1e-5


@pytest.mark.parametrize("chunk", [1, 7, 32, 96])
def test_full_mode_chunked_equals_one_shot(L, port, chunk):
    """test_sparse.cpp:327-338."""
    q, k, v = rin(port, 0, 96, 8, "fp32")
    inp = L.AttentionInput(q, k, v)
    one = L.full_attention(inp)
    pr = L.chunked_prefill(inp, chunk, 1, L.HeadBudget(0, 0), L.PrefillMode.Full,
                           L.PositionMode.Standard, None)
    assert np.abs(pr.result.output - one.output).max() <= 1e-6
    assert np.abs(pr.result.lse - one.lse).max() <= 1e-6


def test_dca_full_budget_equals_remapped_dense(L, port):
    """test_sparse.cpp:406-417."""
    q, k, v = rin(port, 14, 64, 8, "fp32")
    cfg = L.ChunkConfig(16, 48, 16)
    inp = L.AttentionInput(q, k, v)
    pr = L.chunked_prefill(inp, 64, 8, L.HeadBudget(64, 64), L.PrefillMode.Sparse,
                           L.PositionMode.DcaContinuous, cfg)
    dense = L.full_attention(inp, cfg)
    assert row_rel_err(pr.result.output, dense.output) <= 1e-5


def test_cross_chunk_slash_found_only_with_continuous_positions(L, port):
    """test_sparse.cpp:373-404 through the device path."""
    cfg = (32, 128, 32)
    q, k, v = port.make_planted(512, 16, rope_base=1000.0, slash_offsets=[428], strength=12.0,
                                seed=7, dca=cfg, carrier_pairs=[5, 6])
    q, k, v = (rounded(x, "fp32") for x in (q, k, v))
    inp = L.AttentionInput(q, k, v, rope_base=1000.0)
    cont = L.chunked_prefill(inp, 256, 64, L.HeadBudget(0, 2), L.PrefillMode.Sparse,
                             L.PositionMode.DcaContinuous, L.ChunkConfig(*cfg))
    assert 428 in cont.state.selections[1].critical.slashes
    std = L.chunked_prefill(inp, 256, 64, L.HeadBudget(0, 2), L.PrefillMode.Sparse,
                            L.PositionMode.Standard, None)
    assert 428 not in std.state.selections[1].critical.slashes


def test_validation_errors(L, port):
    q, k, v = rin(port, 13, 16, 8, "fp32")
    inp = L.AttentionInput(q, k, v)
    for args, kind in [((0, 1, L.HeadBudget(1, 1), L.PrefillMode.Full, L.PositionMode.Standard,
                         None), "config"),
                       ((8, 0, L.HeadBudget(1, 1), L.PrefillMode.Full, L.PositionMode.Standard,
                         None), "config"),
                       ((4, 8, L.HeadBudget(1, 1), L.PrefillMode.Sparse,
                         L.PositionMode.Standard, None), "config"),
                       ((8, 4, L.HeadBudget(1, 1), L.PrefillMode.Sparse,
                         L.PositionMode.DcaContinuous, None), "config")]:
        with pytest.raises(L.Error) as e:
            L.chunked_prefill(inp, *args)
        assert e.value.kind == kind
    with pytest.raises(L.Error) as e:
        L.estimate_block(q, k, 0, L.PositionMode.Standard, None)
    assert e.value.kind == "config"


# -------------------------------------------------------------------- recall --
def test_attention_recall(L, port):
    rng = np.random.default_rng(3)
    lf = rng.normal(size=1000)
    ls = lf - np.abs(rng.normal(size=1000))
    per_ref, agg_ref = port.attention_recall(ls, lf)
    rep = L.attention_recall(ls, lf)
    assert np.abs(rep.per_query - per_ref).max() <= 1e-6
    assert abs(rep.aggregate - agg_ref) <= 1e-6
    with pytest.raises(L.Error) as e:
        L.attention_recall(lf + 0.1, lf)
    assert e.value.kind == "domain"
    # hand values (test_refine.cpp:31-62)
    assert abs(L.attention_recall([np.log(0.5)], [0.0]).aggregate - 0.5) < 1e-7


def test_measure_budget_recall(L, ref):
    q, k, v = ref.make_planted(128, 16, vertical_columns=[20, 70], slash_offsets=[9],
                               strength=12.0, seed=3)
    q, k, v = (rounded(x, "fp32") for x in (q, k, v))
    exp = ref.lib  # noqa: F841 (reference value below)
    import ctypes as C
    from oracle import _pd
    val = C.c_double()
    qq, kk, vv = (np.ascontiguousarray(x) for x in (q, k, v))
    st = ref.lib.ref_measure_budget_recall(_pd(qq), _pd(kk), _pd(vv), C.c_int64(128),
                                           C.c_int64(16), C.c_double(1e4), C.c_int64(2),
                                           C.c_int64(2), C.c_int64(32), 1, 1, 1, 0,
                                           C.c_double(0.9), C.byref(val))
    assert st == 0
    got = L.measure_budget_recall(L.AttentionInput(q, k, v), L.HeadBudget(2, 2),
                                  L.RecallMeasurement(last_q=32))
    assert abs(got - val.value) <= 1e-5


# ---------------------------------------------------------- multi-head batch --
@pytest.mark.parametrize("precision", ["fp32", "bf16"])
@pytest.mark.parametrize("n", [640, 300, 1])
def test_multihead_gqa_prefill(D, port, precision, n):
    """Batched [n, H, D] entry with GQA (hq=7*hkv): every head equals the single-head
    oracle run on its (q head, kv head) pair."""
    import torch
    hq, hkv, dim = 14, 2, 128
    rng = np.random.default_rng(1)
    q = rounded(rng.standard_normal((n, hq, dim)), precision)
    k = rounded(rng.standard_normal((n, hkv, dim)), precision)
    v = rounded(rng.standard_normal((n, hkv, dim)), precision)
    dt = torch.float32 if precision == "fp32" else torch.bfloat16
    T = lambda x: torch.tensor(x).to(dt).cuda().contiguous()  # noqa: E731
    r = D.chunked_prefill(T(q), T(k), T(v), chunk_len=256, last_q=64, budget=(30, 40),
                          position_mode="dca_continuous", dca=(128, 384, 128), temperature=0.9,
                          return_admitted=True)
    out, lse = r["out"].double().cpu().numpy(), r["lse"].double().cpu().numpy()
    for h in [0, 6, 7, 13]:
        g = h // 7
        o_ref, l_ref, sels = port.chunked_prefill(q[:, h], k[:, g], v[:, g], 256, 64, (30, 40),
                                                  "sparse", 1, (128, 384, 128),
                                                  temperature=0.9)
        for ci, s in enumerate(sels):
            nv, ns = int(r["nv"][ci, h]), int(r["ns"][ci, h])
            assert r["verticals"][ci, h, :nv].tolist() == s.critical.verticals
            assert r["slashes"][ci, h, :ns].tolist() == s.critical.slashes
            t0, t1 = s.begin, s.end
            cnt = sum(len(_adm(s.critical, i)) for i in range(t0, t1))
            assert int(r["admitted"][ci, h]) == cnt
        assert row_rel_err(out[:, h], o_ref) <= TOL[precision]
        assert lse_rel_err(lse[h], l_ref) <= TOL[precision]


def r_crit(r, ci, h, t1):
    from oracle import Critical
    return Critical(r["verticals"][ci, h, :int(r["nv"][ci, h])].tolist(),
                    r["slashes"][ci, h, :int(r["ns"][ci, h])].tolist(), t1)


def _adm(crit, i):
    vs = [x for x in crit.verticals if x <= i]
    ss = [i - d for d in crit.slashes if d <= i]
    row = set(vs) | set(ss)
    return row if row else {i}


# ------------------------------------------------------------ tcgen05 path --
def _mh_inputs(n, hq, hkv, dim, precision, seed, kind="normal"):
    rng = np.random.default_rng(seed)
    q = rng.standard_normal((n, hq, dim))
    k = rng.standard_normal((n, hkv, dim))
    v = rng.standard_normal((n, hkv, dim))
    if kind == "peaked":  # large-logit rows: a few keys aligned with the queries
        k[rng.integers(0, n, n // 16)] *= 6.0
        q *= 1.5
    return (rounded(q, precision), rounded(k, precision), rounded(v, precision))


TC_CASES = [
    # n, hq, hkv, chunk, lq, budget, dca, opts(sink, band), kind, temperature
    (1024, 4, 2, 256, 64, (40, 300), None, (True, True), "normal", 1.0),
    (1536, 6, 2, 512, 64, (100, 200), (256, 768, 256), (True, True), "normal", 0.8),
    (1024, 2, 1, 512, 32, (10, 600), (512, 1024, 512), (False, False), "peaked", 1.0),
    (768, 4, 4, 128, 128, (5, 40), (128, 300, 128), (True, True), "peaked", 1.0),
    (1280, 7, 1, 640, 64, (64, 6), None, (True, False), "normal", 1.0),
    # ragged sequence end (last block / tile partial) under DCA
    (1000, 6, 2, 256, 64, (30, 90), (256, 640, 256), (True, True), "normal", 0.9),
    # budgets beyond the context: every line selected (select k >= n)
    (640, 4, 2, 128, 64, (1000, 1000), None, (True, True), "peaked", 1.0),
    # tiny sequences: one row; a second chunk of two rows; DCA shorter than one chunk pair
    (1, 2, 1, 128, 64, (4, 4), None, (True, True), "normal", 1.0),
    (130, 4, 2, 128, 64, (8, 16), None, (True, True), "normal", 1.0),
    (200, 4, 2, 128, 64, (3, 5), (128, 256, 128), (False, True), "peaked", 0.9),
    # zero budgets: only forced lines, or nothing at all (every row falls back to itself)
    (512, 4, 2, 256, 64, (0, 0), None, (False, False), "normal", 1.0),
    (512, 4, 2, 256, 64, (0, 0), (256, 384, 128), (True, True), "normal", 1.0),
]


@pytest.mark.parametrize("case", TC_CASES)
def test_tc_prefill_matches_oracle(D, port, case):
    """bf16 storage, the tcgen05 tiles + CUDA-core slash path: per head identical
    selections and outputs within 2e-3 of the oracle on the same bf16 values; the TC
    and pure CUDA-core paths agree; admitted-entry counts are exact."""
    import torch
    n, hq, hkv, chunk, lq, bud, dca, (sink, band), kind, temp = case
    q, k, v = _mh_inputs(n, hq, hkv, 128, "bf16", n + hq, kind)
    T = lambda x: torch.tensor(x).to(torch.bfloat16).cuda().contiguous()  # noqa: E731
    opts = D.Options(sink, band, True)
    kw = dict(chunk_len=chunk, last_q=lq, budget=bud, opts=opts, temperature=temp,
              position_mode="dca_continuous" if dca else "standard", dca=dca,
              return_admitted=True)
    r = D.chunked_prefill(T(q), T(k), T(v), kernel_path="tc", **kw)
    rs = D.chunked_prefill(T(q), T(k), T(v), kernel_path="simt", **kw)
    out, lse = r["out"].double().cpu().numpy(), r["lse"].double().cpu().numpy()
    out_s = rs["out"].double().cpu().numpy()
    assert torch.equal(r["admitted"], rs["admitted"])
    assert row_rel_err(out.reshape(n * hq, -1), out_s.reshape(n * hq, -1)) <= 2e-3
    g = hq // hkv
    for h in sorted({0, hq - 1, hq // 2}):
        o_ref, l_ref, sels = port.chunked_prefill(q[:, h], k[:, h // g], v[:, h // g], chunk, lq,
                                                  bud, "sparse", 1 if dca else 0, dca,
                                                  force_sink=sink, force_band=band,
                                                  temperature=temp)
        for ci, s in enumerate(sels):
            gv = r["verticals"][ci, h, :int(r["nv"][ci, h])].tolist()
            gs = r["slashes"][ci, h, :int(r["ns"][ci, h])].tolist()
            if gv != s.critical.verticals or gs != s.critical.slashes:
                # near-tie swap allowed: identical given the device's own fp32 scores
                t0, t1 = s.begin, s.end
                col, sl = D.line_scores(T(q), T(k), q_row0=t0, nq=t1 - t0, nk=t1, last_q=lq,
                                        position_mode="dca_continuous" if dca else "standard",
                                        dca=dca)
                h_k = h // g
                est = port.estimate_block(q[t0:t1, h], k[:t1, h_k], lq, 1 if dca else 0, dca)
                c64, s64 = port.line_scores(est, t1)
                check_selection(port, gv, gs, col[h].double().cpu().numpy(),
                                sl[h].double().cpu().numpy(), c64, s64, t1,
                                min(lq, t1 - t0), bud, sink, band)
                # the oracle's output rows of this chunk under the device's selection
                o_c, l_c = port.sparse_attention(q[:t1, h], k[:t1, h_k], v[:t1, h_k],
                                                 r_crit(r, ci, h, t1), dca=dca,
                                                 temperature=temp)
                o_ref[t0:t1], l_ref[t0:t1] = o_c[t0:t1], l_c[t0:t1]
            cnt = sum(len(_adm(r_crit(r, ci, h, s.end), i)) for i in range(s.begin, s.end))
            assert int(r["admitted"][ci, h]) == cnt
        assert row_rel_err(out[:, h], o_ref) <= 2e-3, h
        assert lse_rel_err(lse[h], l_ref) <= 2e-3, h


@pytest.mark.parametrize("dca", [None, (256, 640, 256)])
@pytest.mark.parametrize("n", [1024, 1, 333])
def test_tc_full_attention(D, port, dca, n):
    import torch
    hq, hkv = 2, 1
    q, k, v = _mh_inputs(n, hq, hkv, 128, "bf16", 3, "peaked")
    T = lambda x: torch.tensor(x).to(torch.bfloat16).cuda().contiguous()  # noqa: E731
    out, lse = D.full_attention(T(q), T(k), T(v), dca=dca, kernel_path="tc", temperature=0.9)
    out, lse = out.double().cpu().numpy(), lse.double().cpu().numpy()
    for h in range(hq):
        o_ref, l_ref = port.full_attention(q[:, h], k[:, 0], v[:, 0], dca=dca, temperature=0.9)
        assert row_rel_err(out[:, h], o_ref) <= 2e-3
        assert lse_rel_err(lse[h], l_ref) <= 2e-3


def test_tc_sparse_attention_custom_positions(D, port):
    import torch
    n = 512
    q, k, v = _mh_inputs(n, 1, 1, 128, "bf16", 9)
    rng = np.random.default_rng(2)
    pq = np.sort(rng.integers(0, 20000, n))
    pk = np.sort(rng.integers(0, 20000, n))
    crit = port.select_critical(port.estimate_block(q[:, 0], k[:, 0], 64), (30, 200), n)
    ref = port.sparse_attention(q[:, 0], k[:, 0], v[:, 0], crit, pos_q=pq, pos_k=pk)
    T = lambda x: torch.tensor(x).to(torch.bfloat16).cuda().contiguous()  # noqa: E731
    Ti = lambda x: torch.tensor(np.asarray(x, np.int32)).cuda().reshape(1, -1)  # noqa: E731
    out, lse = D.sparse_attention(T(q), T(k), T(v), Ti(crit.verticals),
                                  Ti([len(crit.verticals)]).reshape(1),
                                  Ti(crit.slashes), Ti([len(crit.slashes)]).reshape(1),
                                  positions_q=torch.tensor(pq).cuda(),
                                  positions_k=torch.tensor(pk).cuda(), kernel_path="tc")
    assert row_rel_err(out[:, 0].double().cpu().numpy(), ref[0]) <= 2e-3
    assert lse_rel_err(lse[0].double().cpu().numpy(), ref[1]) <= 2e-3


# ------------------------------------------------------------ host entry --
@pytest.mark.parametrize("precision,dca", [("bf16", (256, 768, 256)), ("fp32", None)])
@pytest.mark.parametrize("n", [1280, 1000, 3])
def test_host_entry_equals_device_entry(D, port, precision, dca, n):
    """lcx_chunked_prefill_host (host buffers, chunk-pipelined copies) computes exactly
    what the device entry computes: same kernels, bitwise-equal outputs and selections;
    and the oracle agrees (full, ragged and tiny sequences)."""
    import torch
    hq, hkv = 4, 2
    q, k, v = _mh_inputs(n, hq, hkv, 128, precision, 21)
    dt = torch.float32 if precision == "fp32" else torch.bfloat16
    H = lambda x: torch.tensor(x).to(dt).contiguous().pin_memory()  # noqa: E731
    kw = dict(chunk_len=256, last_q=64, budget=(40, 120), temperature=0.9,
              position_mode="dca_continuous" if dca else "standard", dca=dca)
    rh = D.chunked_prefill_host(H(q), H(k), H(v), return_selections=True, **kw)
    rd = D.chunked_prefill(H(q).cuda(), H(k).cuda(), H(v).cuda(), **kw)
    assert torch.equal(rh["out"], rd["out"].cpu())
    assert torch.equal(rh["lse"], rd["lse"].cpu())
    for key in ("verticals", "nv", "slashes", "ns"):
        assert torch.equal(rh[key], rd[key].cpu()), key
    o_ref, l_ref, _ = port.chunked_prefill(q[:, 3], k[:, 1], v[:, 1], 256, 64, (40, 120),
                                           "sparse", 1 if dca else 0, dca, temperature=0.9)
    assert row_rel_err(rh["out"][:, 3].double().numpy(), o_ref) <= TOL[precision]


# ------------------------------------------------------- KV-line sharding --
@pytest.mark.parametrize("shards", [2, 3])
@pytest.mark.parametrize("path,precision,dca", [("tc", "bf16", (256, 768, 256)),
                                                ("simt", "fp32", None)])
@pytest.mark.parametrize("n", [1024, 200])
def test_line_sharded_prefill_merges_to_unsharded(D, port, shards, path, precision, dca, n):
    """North star (e): every shard attends over its part of the selected lines; the LSE
    merge of the partials (on-device merge of stacked partials, and the collective path's
    per-shard scaling + sum) equals the unsharded operator and the oracle; admitted
    counts add up (rank 0 reports the exact count, sparse.cpp:115-119)."""
    import torch
    hq, hkv = 4, 2
    q, k, v = _mh_inputs(n, hq, hkv, 128, precision, 31, "peaked")
    dt = torch.float32 if precision == "fp32" else torch.bfloat16
    T = lambda x: torch.tensor(x).to(dt).cuda().contiguous()  # noqa: E731
    qt, kt, vt = T(q), T(k), T(v)
    kw = dict(chunk_len=256, last_q=64, budget=(40, 200), temperature=0.9, kernel_path=path,
              position_mode="dca_continuous" if dca else "standard", dca=dca,
              return_admitted=True)
    full = D.chunked_prefill(qt, kt, vt, **kw)
    parts = [D.chunked_prefill(qt, kt, vt, shard=(r, shards), **kw) for r in range(shards)]
    for p in parts:  # every shard logs the full selection
        assert torch.equal(p["verticals"], full["verticals"])
        assert torch.equal(p["slashes"], full["slashes"])
    assert int(sum(p["admitted"].sum() for p in parts)) == int(full["admitted"].sum())
    o = torch.stack([p["out"] for p in parts]).reshape(shards, n * hq, 128)
    ls = torch.stack([p["lse"] for p in parts]).transpose(1, 2).reshape(shards, n * hq)
    mo, ml = D.lse_merge(o.contiguous(), ls.contiguous())
    mo = mo.reshape(n, hq, 128).double().cpu().numpy()
    ml = ml.reshape(n, hq).t().double().cpu().numpy()
    tol = TOL[precision]
    ref_o, ref_l = full["out"].double().cpu().numpy(), full["lse"].double().cpu().numpy()
    assert row_rel_err(mo.reshape(n * hq, -1), ref_o.reshape(n * hq, -1)) <= tol
    assert lse_rel_err(ml, ref_l) <= tol
    # collective form: scale each partial by exp(lse_g - lse_tot), then sum over shards
    lse_all = torch.stack([p["lse"] for p in parts]).contiguous()
    acc = torch.zeros_like(parts[0]["out"])
    for p in parts:
        tot = D.lse_scale_partial(p["out"], p["lse"], lse_all)
        acc += p["out"]
    assert row_rel_err(acc.double().cpu().numpy().reshape(n * hq, -1),
                       ref_o.reshape(n * hq, -1)) <= tol
    assert lse_rel_err(tot.double().cpu().numpy(), ref_l) <= tol
    o_ref, l_ref, _ = port.chunked_prefill(q[:, 1], k[:, 0], v[:, 0], 256, 64, (40, 200),
                                           "sparse", 1 if dca else 0, dca, temperature=0.9)
    assert row_rel_err(mo[:, 1], o_ref) <= tol


@pytest.mark.parametrize("geom", [(28, 4), (40, 8)])
@pytest.mark.parametrize("dca", [None, (1024, 3072, 1024)])
def test_sharded_estimator_selections_bitwise_g_invariant(D, geom, dca):
    """North star (e), sharded estimator: the select phase of each of G = 2 / 4 / 8 ranks
    (its head pairs only, run one after the other on this GPU) writes exactly its heads'
    slots, and the union of the G shards' lists is bitwise the unsharded selection (every
    chunk, every head); the attend phase over the union equals the unsharded operator
    bitwise (same lists, same kernels)."""
    import torch
    from paper_2501_15383_b200 import shard as SH
    from paper_2501_15383_b200.synth import make_qkv
    hq, hkv = geom
    n = 4096
    q, k, v = make_qkv(n, hq, hkv, kind="planted", seed=5, device="cuda", rope_base=1e6)
    kw = dict(chunk_len=1024, last_q=64, budget=(48, 160), temperature=0.9, rope_base=1e6,
              position_mode="dca_continuous" if dca else "standard", dca=dca)
    full = D.chunked_prefill(q, k, v, **kw)
    keys = ("verticals", "nv", "slashes", "ns")
    for G in (2, 4, 8):
        union = {x: torch.zeros_like(full[x]) for x in keys}
        for r, (h0, h1) in enumerate(SH.est_head_ranges(hq, hkv, G)):
            if h1 <= h0:
                continue
            sel = {x: torch.full_like(full[x], -7) for x in keys}
            D.chunked_prefill(q, k, v, phase="select", est_heads=(h0, h1), selections=sel, **kw)
            for x in keys:
                assert (sel[x][:, :h0] == -7).all() and (sel[x][:, h1:] == -7).all()
                union[x][:, h0:h1] = sel[x][:, h0:h1]
        for x in keys:
            assert torch.equal(union[x], full[x]), (G, x)
    att = D.chunked_prefill(q, k, v, phase="attend", selections=union, **kw)
    assert torch.equal(att["out"], full["out"]) and torch.equal(att["lse"], full["lse"])


def test_seq_prefill_one_gpu_emulation(D):
    """The seq strategy's merge on the device (lcx_stream_wait_chunk + lse_scale_partial)
    for G = 2 shards emulated in one process: a trivial process group of size 1 cannot run
    it, so each 'rank' here runs the attend phase of its line shard and the per-chunk
    merge is formed as seq_prefill forms it (all_gather = stack, reduce_scatter = sum +
    slice); the merged rows equal the unsharded operator within the bf16 tolerance."""
    import torch
    from paper_2501_15383_b200 import shard as SH
    from paper_2501_15383_b200.synth import make_qkv
    n, hq, hkv, G, L = 4096, 28, 4, 2, 1024
    q, k, v = make_qkv(n, hq, hkv, kind="planted", seed=6, device="cuda", rope_base=1e6)
    kw = dict(chunk_len=L, last_q=64, budget=(48, 160), temperature=0.9, rope_base=1e6,
              position_mode="dca_continuous", dca=(2048, 4096, 2048))
    full = D.chunked_prefill(q, k, v, **kw)
    sel = {x: full[x] for x in ("verticals", "nv", "slashes", "ns")}
    parts = []
    for r in range(G):
        out = torch.empty((n, hq, 128), device="cuda")
        lse = torch.empty((hq, n), device="cuda")
        D.chunked_prefill(q, k, v, phase="attend", selections=sel, shard=(r, G),
                          record_chunk_events=True, out=out, lse=lse, **kw)
        side = torch.cuda.Stream()
        for c in range(n // L):  # every chunk's event is recorded and waitable
            D.stream_wait_chunk(c, side)
        torch.cuda.current_stream().wait_stream(side)
        parts.append((out, lse))
    for r in range(G):
        rows = []
        for c, (t0, t1) in enumerate(SH.chunk_bounds(n, L)):
            lse_all = torch.stack([p[1][:, t0:t1] for p in parts]).contiguous()
            acc = torch.zeros((t1 - t0, hq, 128), device="cuda")
            for out, lse in parts:
                o_c = out[t0:t1].clone()
                D.lse_scale_partial(o_c, lse[:, t0:t1].contiguous(), lse_all)
                acc += o_c
            a, b = SH.seq_row_ranges(n, L, G, r)[c]
            rows.append(acc[a - t0:b - t0])
        got = torch.cat(rows).double().cpu().numpy()
        ref = torch.cat([full["out"][a:b] for a, b in SH.seq_row_ranges(n, L, G, r)])
        ref = ref.double().cpu().numpy()
        assert row_rel_err(got.reshape(-1, 128), ref.reshape(-1, 128)) <= 2e-3


# ------------------------------------------------------------- recall check --
@pytest.mark.parametrize("precision,dca", [("bf16", (256, 768, 256)), ("fp32", None),
                                           ("bf16", None)])
@pytest.mark.parametrize("n,lq", [(1024, 64), (1000, 64), (40, 64), (700, 200)])
def test_prefill_recall_check(D, port, precision, dca, n, lq):
    """North star (d): the operator's recall check (dense LSE of each chunk's last lastQ
    rows vs the sparse LSE) equals the reference's attention_recall on the oracle's
    sparse and dense LSE of the same rows (refine.cpp:51-72); full budget -> recall 1."""
    import torch
    hq, hkv, chunk = 2, 1, 256
    q, k, v = _mh_inputs(n, hq, hkv, 128, precision, 41, "peaked")
    dt = torch.float32 if precision == "fp32" else torch.bfloat16
    T = lambda x: torch.tensor(x).to(dt).cuda().contiguous()  # noqa: E731
    kw = dict(chunk_len=chunk, last_q=lq, temperature=0.9,
              position_mode="dca_continuous" if dca else "standard", dca=dca)
    r = D.chunked_prefill(T(q), T(k), T(v), budget=(8, 16), return_recall=True, **kw)
    rec = r["recall"].double().cpu().numpy()
    tol = 1e-4 if precision == "fp32" else 4e-3
    for h in range(hq):
        o_s, l_s, _ = port.chunked_prefill(q[:, h], k[:, 0], v[:, 0], chunk, lq, (8, 16),
                                           "sparse", 1 if dca else 0, dca, temperature=0.9)
        o_f, l_f, _ = port.chunked_prefill(q[:, h], k[:, 0], v[:, 0], chunk, lq, (8, 16),
                                           "full", 1 if dca else 0, dca, temperature=0.9)
        for ci in range(-(-n // chunk)):  # the last B = min(lastQ, rows) rows of each chunk
            t1 = min(n, (ci + 1) * chunk)
            rows = slice(t1 - min(lq, t1 - ci * chunk), t1)
            per, agg = port.attention_recall(l_s[rows], l_f[rows], slack=1e-9)
            assert abs(rec[ci, h] - agg) <= tol, (ci, h, rec[ci, h], agg)
    full = D.chunked_prefill(T(q), T(k), T(v), budget=(n, n), return_recall=True, **kw)
    assert float(full["recall"].min()) >= 1.0 - tol


@pytest.mark.gpu
def test_kernel_path_stat_reports_auto_fallback():
    """LCX_PATH_AUTO on bf16 runs the tcgen05 kernels on 128-aligned chunks and reports the
    CUDA-core fallback otherwise (lcx_prefill_stats.tc_path), never silently."""
    import torch
    from paper_2501_15383_b200 import device as D
    from paper_2501_15383_b200._lib import context
    ctx = context(0)
    g = torch.Generator(device="cuda").manual_seed(5)
    q, k, v = (torch.randn((512, h, 128), generator=g, device="cuda").to(torch.bfloat16)
               for h in (2, 1, 1))
    D.chunked_prefill(q, k, v, chunk_len=256, last_q=64, budget=(16, 32), ctx=ctx)
    torch.cuda.synchronize()
    assert ctx.stats()["tc_path"] == 1
    D.chunked_prefill(q, k, v, chunk_len=200, last_q=64, budget=(16, 32), ctx=ctx)
    torch.cuda.synchronize()
    assert ctx.stats()["tc_path"] == 0


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["device", "host"])
def test_chunk_range_matches_full_prefill(kind):
    """chunks=(c0, c1) computes exactly the full run's rows of chunks [c0, c1) (bitwise),
    selections and admitted counts included, and leaves the other rows untouched -- the
    multi-GPU plan that splits a query head's chunks over two ranks relies on it."""
    import torch
    from paper_2501_15383_b200 import device as D
    g = torch.Generator(device="cuda").manual_seed(11)
    n, L = 2048, 512
    q, k, v = (torch.randn((n, h, 128), generator=g, device="cuda").to(torch.bfloat16)
               for h in (4, 2, 2))
    kw = dict(chunk_len=L, last_q=64, budget=(32, 96), position_mode="dca_continuous",
              dca=(1024, 2048, 1024), rope_base=1e4)
    full = D.chunked_prefill(q, k, v, return_admitted=True, **kw)
    torch.cuda.synchronize()
    c0, c1 = 1, 3
    if kind == "device":
        out = torch.full((n, 4, 128), 7.0, device="cuda")
        lse = torch.full((4, n), 7.0, device="cuda")
        part = D.chunked_prefill(q, k, v, out=out, lse=lse, return_admitted=True,
                                 chunks=(c0, c1), **kw)
        torch.cuda.synchronize()
        assert torch.equal(part["admitted"][c0:c1], full["admitted"][c0:c1])
        assert int(part["admitted"][:c0].sum()) == 0 and int(part["admitted"][c1:].sum()) == 0
        o, l_ = out.cpu(), lse.cpu()
    else:
        hq_, hk_, hv_ = (x.cpu().pin_memory() for x in (q, k, v))
        out = torch.full((n, 4, 128), 7.0).pin_memory()
        lse = torch.full((4, n), 7.0).pin_memory()
        part = D.chunked_prefill_host(hq_, hk_, hv_, out=out, lse=lse, return_selections=True,
                                      chunks=(c0, c1), **kw)
        o, l_ = out, lse
    r0, r1 = c0 * L, c1 * L
    assert torch.equal(o[r0:r1], full["out"][r0:r1].cpu())
    assert torch.equal(l_[:, r0:r1], full["lse"][:, r0:r1].cpu())
    assert torch.all(o[:r0] == 7.0) and torch.all(o[r1:] == 7.0)
    for key in ("verticals", "nv", "slashes", "ns"):
        assert torch.equal(part[key][c0:c1].cpu(), full[key][c0:c1].cpu()), key


@pytest.mark.gpu
def test_balanced_plan_parts_match_full_prefill():
    """The cost-balanced multi-GPU plan (shard.balanced_plan, auto at G > 1): calibrated
    per-(KV head, chunk) costs, every rank's parts run as chunk-ranged prefills over their
    KV heads -- together they reproduce the single-GPU layer bitwise, every (head, row) once."""
    import torch
    from paper_2501_15383_b200 import device as D, shard as SH
    from paper_2501_15383_b200._lib import context
    g = torch.Generator(device="cuda").manual_seed(12)
    n, L, hq, hkv = 2048, 512, 6, 3
    q = torch.randn((n, hq, 128), generator=g, device="cuda").to(torch.bfloat16)
    k, v = (torch.randn((n, hkv, 128), generator=g, device="cuda").to(torch.bfloat16)
            for _ in range(2))
    kw = dict(chunk_len=L, last_q=64, budget=(32, 96), position_mode="dca_continuous",
              dca=(1024, 2048, 1024), rope_base=1e4)
    full = D.chunked_prefill(q, k, v, return_admitted=True, **kw)
    torch.cuda.synchronize()
    costs = SH.calibrate(q, k, v, context(0), **kw)
    assert len(costs) == hkv and all(len(r) == n // L and min(r) > 0 for r in costs)
    covered = torch.zeros((n, hq), dtype=torch.int32)
    adm_total = 0
    for world in (2, 4):
        covered.zero_()
        adm_total = 0
        for rank in range(world):
            p = SH.balanced_plan(costs, n, hq, hkv, world, rank)
            qs, ks, vs = SH.take(p, q, k, v)
            r = SH.prefill(p, qs, ks, vs, return_admitted=True, **kw)
            torch.cuda.synchronize()
            adm_total += int(r["admitted"].sum())
            for (a, b, c0, c1), part in zip(p.segments, r["segments"]):
                r0, r1 = (c0 or 0) * L, n if c1 is None else c1 * L
                h0, h1 = a * 2, b * 2
                assert torch.equal(part["out"][r0:r1], full["out"][r0:r1, h0:h1])
                assert torch.equal(part["lse"][:, r0:r1], full["lse"][h0:h1, r0:r1])
                covered[r0:r1, h0:h1] += 1
            assert p.notes["stats"]["chunks"] > 0
        assert torch.all(covered == 1)
        assert adm_total == int(full["admitted"].sum())
