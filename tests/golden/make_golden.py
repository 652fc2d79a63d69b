"""Generate the golden fixtures under tests/golden/ from the REFERENCE itself.

Run here (where /root/reference exists), after `make -C oracle`:

    python tests/golden/make_golden.py

It drives the unmodified reference library (oracle/_ref/liblongctx_ref.so) and writes:

  sparsity_example.json  replay of `longctx sparsity --config proj/configs/example.json`
                          (harness.cpp:328-441); asserted equal to the committed
                          proj/out/sparsity/{critical_set,prefill_selections}.json and
                          sparsity_checks.csv values before writing.
  sparsity_dca.json      the same replay on proj/configs/dca_sparsity.json (no committed
                          outputs in the reference; values from the reference library).
  kat_hashes.json        sha256 of reference outputs (estimate/select/sparse/chunked/dca/
                          full attention) on seeded inputs; the port must reproduce them
                          bit-for-bit (tests/test_oracle_pin.py).

The GPU box never runs this script (it has no /root/reference); it only reads the
committed JSON.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from oracle import Oracle, Rng  # noqa: E402

REF_OUT = "/root/reference/proj/out/sparsity"


def replay_spec(port: Oracle, ref: Oracle, seed, n, dim, chunk_len, last_q, budget, pv, ps,
                strength, dca_mode, chunk_cfg, rope_base=1e4):
    """Planted-spec construction of run_sparsity (harness.cpp:332-372)."""
    ms = ref.lib.ref_module_seed(seed, b"vertical-slash")
    spec_seed = Rng(port, ms).next_u64()
    lo_v = min(64, n // 4)
    vcols = [lo_v + i * max(1, (n // 2 - lo_v) // max(1, pv)) for i in range(pv)]
    s, c, w = chunk_cfg
    if dca_mode:
        lo_s = max(1, w // 2)
        hi_s = max(lo_s + 1, w)
    else:
        lo_s = min(last_q, n // 4)
        hi_s = n // 2
    soffs = sorted(set(min(n - 1, lo_s + i * max(1, (hi_s - lo_s) // max(1, ps)))
                       for i in range(ps)))
    return dict(n=n, dim=dim, rope_base=rope_base, vertical_columns=vcols, slash_offsets=soffs,
                vertical_strength=strength, slash_strength=1.6 * strength, seed=int(spec_seed),
                dca=list(chunk_cfg) if dca_mode else None)


def run_replay(ref: Oracle, spec, chunk_len, last_q, budget, dca_mode, chunk_cfg):
    q, k, v = ref.make_planted(spec["n"], spec["dim"], rope_base=spec["rope_base"],
                               vertical_columns=spec["vertical_columns"],
                               slash_offsets=spec["slash_offsets"],
                               vertical_strength=spec["vertical_strength"],
                               slash_strength=spec["slash_strength"], seed=spec["seed"],
                               dca=tuple(spec["dca"]) if spec["dca"] else None)
    n = spec["n"]
    pm = 1 if dca_mode else 0
    cfg = tuple(chunk_cfg) if dca_mode else None
    est = ref.estimate_block(q, k, last_q, pm, cfg, spec["rope_base"])
    crit = ref.select_critical(est, budget, n)
    full = ref.full_attention(q, k, v, rope_base=spec["rope_base"], dca=cfg)
    sp = ref.sparse_attention(q, k, v, crit, rope_base=spec["rope_base"], dca=cfg)
    _, recall = ref.attention_recall(sp[1], full[1])
    dens = ref.density(crit.verticals, crit.slashes, n)
    _, _, sels = ref.chunked_prefill(q, k, v, chunk_len, last_q, budget, "sparse", pm, cfg,
                                     rope_base=spec["rope_base"])
    return dict(
        critical={"contextLength": n, "verticals": [int(x) for x in crit.verticals],
                  "slashes": [int(x) for x in crit.slashes]},
        recall=recall, density=dens,
        selections=[{"chunk": s.chunk_index, "begin": s.begin, "end": s.end,
                     "critical": {"contextLength": s.critical.context_length,
                                  "verticals": [int(x) for x in s.critical.verticals],
                                  "slashes": [int(x) for x in s.critical.slashes]}}
                    for s in sels],
        input_sha256=sha(q, k, v))


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a, dtype=np.float64).tobytes())
    return h.hexdigest()


def main():
    port, ref = Oracle("port"), Oracle("reference")

    # --- example.json: seed 42, n 1024, D 128, chunk {64, 128}, budget (2,2) ---------
    ex = dict(seed=42, n=1024, dim=128, chunk_len=256, last_q=64, budget=(2, 2), pv=2, ps=2,
              strength=80.0, dca_mode=False, chunk_cfg=(64, 128, 64))
    spec = replay_spec(port, ref, **ex)
    res = run_replay(ref, spec, ex["chunk_len"], ex["last_q"], ex["budget"], False,
                     ex["chunk_cfg"])
    committed_crit = json.load(open(os.path.join(REF_OUT, "critical_set.json")))
    committed_sel = json.load(open(os.path.join(REF_OUT, "prefill_selections.json")))
    assert res["critical"]["verticals"] == committed_crit["verticals"]
    assert res["critical"]["slashes"] == committed_crit["slashes"]
    assert [s["critical"] for s in res["selections"]] == \
        [s["critical"] for s in committed_sel["selections"]]
    assert repr(res["recall"]) == "0.9994254672010002", res["recall"]
    assert repr(res["density"]) == "0.12907393292682925", res["density"]
    json.dump(dict(source="proj/configs/example.json replayed through harness.cpp:328-441; "
                          "equals proj/out/sparsity/* (configHash 6ae0a4a434c413c7)",
                   config=dict(ex, budget=list(ex["budget"]), chunk_cfg=list(ex["chunk_cfg"])),
                   spec=spec, expected=res),
              open(os.path.join(HERE, "sparsity_example.json"), "w"), indent=1)

    # --- dca_sparsity.json: seed 3, chunk {128, 512, w=128}, dcaContinuous ----------
    dc = dict(seed=3, n=1024, dim=128, chunk_len=256, last_q=64, budget=(2, 2), pv=2, ps=2,
              strength=80.0, dca_mode=True, chunk_cfg=(128, 512, 128))
    spec = replay_spec(port, ref, **dc)
    res = run_replay(ref, spec, dc["chunk_len"], dc["last_q"], dc["budget"], True,
                     dc["chunk_cfg"])
    json.dump(dict(source="proj/configs/dca_sparsity.json replayed through harness.cpp:328-441 "
                          "on the reference library (no committed reference output)",
                   config=dict(dc, budget=list(dc["budget"]), chunk_cfg=list(dc["chunk_cfg"])),
                   spec=spec, expected=res),
              open(os.path.join(HERE, "sparsity_dca.json"), "w"), indent=1)

    # --- known-answer hashes on seeded random inputs ----------------------------------
    kat = []
    for seed, n, dim, lq, bud, pm, cfg, chunk in [
            (1, 64, 8, 16, (4, 4), 0, None, 32), (2, 200, 16, 32, (5, 7), 0, None, 64),
            (3, 256, 32, 64, (8, 8), 1, (32, 96, 32), 128), (4, 300, 16, 64, (3, 5), 1,
                                                            (64, 128, 64), 100),
            (5, 512, 128, 64, (16, 32), 0, None, 256)]:
        q, k, v = port.random_input(seed, n, dim)
        est = ref.estimate_block(q[n - chunk:], k, lq, pm, cfg)
        crit = ref.select_critical(est, bud, n)
        sp = ref.sparse_attention(q, k, v, crit, dca=cfg)
        out, lse, sels = ref.chunked_prefill(q, k, v, chunk, lq, bud, "sparse", pm, cfg)
        full = ref.full_attention(q, k, v, dca=cfg)
        entry = dict(seed=seed, n=n, dim=dim, last_q=lq, budget=list(bud), pos_mode=pm,
                     cfg=list(cfg) if cfg else None, chunk_len=chunk,
                     input=sha(q, k, v), est=sha(est),
                     verticals=[int(x) for x in crit.verticals],
                     slashes=[int(x) for x in crit.slashes],
                     sparse=sha(*sp), prefill=sha(out, lse), full=sha(*full),
                     selections=[[int(x) for x in s.critical.verticals] +
                                 [-1] + [int(x) for x in s.critical.slashes] for s in sels])
        if cfg:
            entry["dca_attention"] = sha(*ref.dca_attention(q, k, v, cfg, 4.0))
        kat.append(entry)
    json.dump(dict(source="reference library outputs (oracle/_ref) on "
                          "testutil::random_input(seed) inputs", cases=kat,
                   yarn={str(s): ref.yarn_temperature(s) for s in (1.0, 2.0, 4.0, 8.0)}),
              open(os.path.join(HERE, "kat_hashes.json"), "w"), indent=1)
    print("golden fixtures written")


if __name__ == "__main__":
    main()
