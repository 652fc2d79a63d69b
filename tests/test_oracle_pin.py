"""Pin the CPU oracle (oracle/longctx_oracle.c) before trusting it.

1. Against the committed golden fixtures (tests/golden/*.json, generated from the
   reference library by tests/golden/make_golden.py; the example fixture equals the
   reference's own committed proj/out/sparsity/* reports) -- runs everywhere.
2. Bit-for-bit against the reference library itself (oracle/_ref) when it was built
   here (skipped on the GPU box, where /root/reference does not exist).
"""
import hashlib
import json
import os

import numpy as np
import pytest

from helpers import rounded  # noqa: F401

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a, dtype=np.float64).tobytes())
    return h.hexdigest()


def planted_from_spec(o, spec):
    return o.make_planted(spec["n"], spec["dim"], rope_base=spec["rope_base"],
                          vertical_columns=spec["vertical_columns"],
                          slash_offsets=spec["slash_offsets"],
                          vertical_strength=spec["vertical_strength"],
                          slash_strength=spec["slash_strength"], seed=spec["seed"],
                          dca=tuple(spec["dca"]) if spec["dca"] else None)


@pytest.mark.parametrize("name", ["sparsity_example.json", "sparsity_dca.json"])
def test_port_reproduces_sparsity_goldens(port, name):
    g = json.load(open(os.path.join(GOLD, name)))
    cfg, spec, exp = g["config"], g["spec"], g["expected"]
    q, k, v = planted_from_spec(port, spec)
    assert sha(q, k, v) == exp["input_sha256"]
    dca = tuple(cfg["chunk_cfg"]) if cfg["dca_mode"] else None
    pm = 1 if cfg["dca_mode"] else 0
    est = port.estimate_block(q, k, cfg["last_q"], pm, dca, spec["rope_base"])
    crit = port.select_critical(est, tuple(cfg["budget"]), spec["n"])
    assert crit.verticals == exp["critical"]["verticals"]
    assert crit.slashes == exp["critical"]["slashes"]
    full = port.full_attention(q, k, v, rope_base=spec["rope_base"], dca=dca)
    sp = port.sparse_attention(q, k, v, crit, rope_base=spec["rope_base"], dca=dca)
    _, recall = port.attention_recall(sp[1], full[1])
    assert recall == exp["recall"]  # bitwise
    assert port.density(crit.verticals, crit.slashes, spec["n"]) == exp["density"]
    _, _, sels = port.chunked_prefill(q, k, v, cfg["chunk_len"], cfg["last_q"],
                                      tuple(cfg["budget"]), "sparse", pm, dca,
                                      rope_base=spec["rope_base"])
    assert [dict(verticals=s.critical.verticals, slashes=s.critical.slashes) for s in sels] == \
        [dict(verticals=s["critical"]["verticals"], slashes=s["critical"]["slashes"])
         for s in exp["selections"]]


def test_example_golden_matches_reference_reports():
    """The fixture values are the reference's committed report values."""
    g = json.load(open(os.path.join(GOLD, "sparsity_example.json")))
    assert repr(g["expected"]["recall"]) == "0.9994254672010002"
    assert repr(g["expected"]["density"]) == "0.12907393292682925"
    assert g["expected"]["critical"]["verticals"] == [0, 64, 288]
    assert g["expected"]["selections"][0]["critical"]["verticals"] == [0, 64, 171]


def test_port_reproduces_kat_hashes(port):
    g = json.load(open(os.path.join(GOLD, "kat_hashes.json")))
    for c in g["cases"]:
        q, k, v = port.random_input(c["seed"], c["n"], c["dim"])
        assert sha(q, k, v) == c["input"]
        cfg = tuple(c["cfg"]) if c["cfg"] else None
        n, chunk = c["n"], c["chunk_len"]
        est = port.estimate_block(q[n - chunk:], k, c["last_q"], c["pos_mode"], cfg)
        assert sha(est) == c["est"], c
        crit = port.select_critical(est, tuple(c["budget"]), n)
        assert crit.verticals == c["verticals"] and crit.slashes == c["slashes"]
        assert sha(*port.sparse_attention(q, k, v, crit, dca=cfg)) == c["sparse"]
        out, lse, sels = port.chunked_prefill(q, k, v, chunk, c["last_q"], tuple(c["budget"]),
                                              "sparse", c["pos_mode"], cfg)
        assert sha(out, lse) == c["prefill"]
        assert [s.critical.verticals + [-1] + s.critical.slashes for s in sels] == c["selections"]
        assert sha(*port.full_attention(q, k, v, dca=cfg)) == c["full"]
        if cfg:
            assert sha(*port.dca_attention(q, k, v, cfg, 4.0)) == c["dca_attention"]
    for s, t in g["yarn"].items():
        assert port.yarn_temperature(float(s)) == t


def test_dca_hand_values(port):
    """test_dca.cpp hand values: cfg {6, 10, 4}: (7,5)->2, (13,0)->9, (11,2)->7 ..."""
    # dca_relative(i, j) with s=6, c=10
    assert port.dca_relative(7, 5, 6, 10) == 2
    assert port.dca_relative(13, 0, 6, 10) == 9
    assert port.dca_relative(11, 2, 6, 10) == 7
    assert abs(port.yarn_temperature(4.0) - 0.771321) < 1e-6
    assert abs(port.yarn_temperature(8.0) - 0.685341) < 1e-6


def test_density_worked_example(port):
    """test_sparse.cpp:260-272: forced-only, n=1024, lastQ=64."""
    est = np.zeros((64, 1024))
    crit = port.select_critical(est, (0, 0), 1024)
    assert crit.verticals == [0] and crit.slashes == list(range(64))
    expected = sum(1024 - d for d in range(64)) + (1024 - 64)
    assert port.admitted_count(crit.verticals, crit.slashes, 1024) == expected
    assert abs(expected / 524800.0 - 0.1229) < 1e-3


def test_ties_break_to_smaller_index(port):
    est = np.zeros((1, 6))
    est[0, 2] = 0.4
    est[0, 5] = 0.4
    est[0, 0] = 0.2
    crit = port.select_critical(est, (1, 0), 6, False, False, True)
    assert crit.verticals == [2] and crit.slashes == []


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_port_bitwise_equals_reference(port, ref, seed):
    rng = np.random.default_rng(seed)
    n, dim = int(rng.integers(40, 300)), int(rng.choice([8, 16, 32]))
    q, k, v = port.random_input(seed * 7, n, dim)
    for pm, cfg in [(0, None), (1, (16, 48, 16)), (1, (6, 10, 4))]:
        chunk = int(rng.integers(16, n + 1))
        lq = int(rng.integers(1, chunk + 1))
        bud = (int(rng.integers(0, 10)), int(rng.integers(0, 10)))
        a = port.chunked_prefill(q, k, v, chunk, lq, bud, "sparse", pm, cfg)
        b = ref.chunked_prefill(q, k, v, chunk, lq, bud, "sparse", pm, cfg)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
        for x, y in zip(a[2], b[2]):
            assert x.critical.verticals == y.critical.verticals
            assert x.critical.slashes == y.critical.slashes
        if cfg:
            assert np.array_equal(port.dca_attention(q, k, v, cfg, 4.0)[0],
                                  ref.dca_attention(q, k, v, cfg, 4.0)[0])
    for dca in [None, (32, 128, 32)]:
        a = port.make_planted(256, 16, rope_base=1000.0, vertical_columns=[30], slash_offsets=[70],
                              strength=12.0, seed=seed, dca=dca, carrier_pairs=[5, 6])
        b = ref.make_planted(256, 16, rope_base=1000.0, vertical_columns=[30], slash_offsets=[70],
                             strength=12.0, seed=seed, dca=dca, carrier_pairs=[5, 6])
        assert all(np.array_equal(x, y) for x, y in zip(a, b))


def test_errors_match_reference_kinds(port, ref):
    q, k, v = port.random_input(1, 16, 8)
    from oracle import OracleError
    for o in (port, ref):
        with pytest.raises(OracleError) as e:
            o.chunked_prefill(q, k, v, 0, 1, (1, 1), "full")
        assert e.value.kind == "config"
        with pytest.raises(OracleError) as e:
            o.chunked_prefill(q, k, v, 4, 8, (1, 1), "sparse")
        assert e.value.kind == "config"
        with pytest.raises(OracleError) as e:
            o.estimate_block(q, k, 0)
        assert e.value.kind == "config"


@pytest.mark.parametrize("dca", [None, (64, 192, 64)])
def test_row_list_oracle_equals_whole_sequence_oracle(port, dca):
    """lco_attention_row_list (row-sampled parity at 128K-1M) computes exactly the rows
    sparse_attention / full_attention compute (same per-row arithmetic)."""
    q, k, v = port.random_input(3, 300, 16)
    crit = port.select_critical(port.estimate_block(q, k, 64), (10, 20), 300)
    rows = [0, 5, 150, 299]
    for c in (crit, None):
        fo, fl = (port.sparse_attention(q, k, v, c, dca=dca, temperature=0.8) if c else
                  port.full_attention(q, k, v, dca=dca, temperature=0.8))
        ro, rl = port.attention_rows(q, k, v, rows, c, dca=dca, temperature=0.8)
        assert np.array_equal(ro, fo[rows]) and np.array_equal(rl, fl[rows])


@pytest.mark.parametrize("pm,cfg", [(0, None), (1, (32, 96, 32)), (1, (6, 10, 4))])
def test_fast_estimator_restatement_pinned(port, pm, cfg):
    """oracle.estimate_probs_fast / line_scores_fast (the large-scale parity checker) equal
    the per-entry C restatement of estimate_block + select_critical's line sums."""
    from oracle import estimate_probs_fast, line_scores_fast
    rng = np.random.default_rng(7)
    n, dim, B = 300, 128, 64
    q, k = rng.standard_normal((n, dim)), rng.standard_normal((n, dim))
    ref = port.estimate_block(q[n - 100:], k, B, pm, cfg, 1e4)
    got = estimate_probs_fast(q[n - B:], k, pm, cfg[1] if cfg else 0, 1e4)
    assert np.abs(got - ref).max() <= 1e-13
    c1, s1 = port.line_scores(ref, n)
    c2, s2 = line_scores_fast(got)
    assert np.abs(c1 - c2).max() <= 1e-12 and np.abs(s1 - s2).max() <= 1e-12
