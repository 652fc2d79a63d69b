"""The C++ drop-in (include/longctx_b200.hpp over liblongctx_b200.so), driven by a C++
program written against the reference's API (tests/cpp/dropin_parity.cpp):

  * CPU: it compiles and links against the library, and the host-side validation
    throws the reference's error kinds (and kind "cuda" -- never a CPU fallback --
    when there is no device);
  * GPU: its results equal the oracle's on the same inputs (selections exactly,
    given the device's own fp32 scores; outputs within the fp32 tolerance).
"""
import os
import struct
import subprocess

import numpy as np
import pytest

from oracle import Critical

from helpers import TOL, lse_rel_err, rounded, row_rel_err

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "dropin_parity.cpp")
BIN = os.path.join(ROOT, "tests", "cpp", "dropin_parity")


def build_binary():
    from paper_2501_15383_b200 import _lib
    lib_dir = os.path.dirname(_lib.LIB_PATH)
    if os.path.exists(BIN) and os.path.getmtime(BIN) >= max(os.path.getmtime(SRC),
                                                            os.path.getmtime(_lib.LIB_PATH)):
        return BIN
    tmp = f"{BIN}.{os.getpid()}.tmp"
    subprocess.run(["g++", "-std=c++20", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"), SRC,
                    "-L", lib_dir, "-llongctx_b200", f"-Wl,-rpath,{lib_dir}", "-o", tmp],
                   check=True)
    os.replace(tmp, BIN)  # atomic: parallel workers never exec a half-written binary
    return BIN


def test_dropin_compiles_and_validates_like_the_reference():
    import torch
    env = dict(os.environ)
    if not torch.cuda.is_available():
        env["LCX_EXPECT_NO_GPU"] = "1"
    r = subprocess.run([build_binary(), "--errors"], capture_output=True, text=True, env=env)
    assert r.returncode == 0, r.stdout + r.stderr


def _read_records(path):
    recs = []
    with open(path, "rb") as f:
        while True:
            h = f.read(8)
            if not h:
                break
            (cnt,) = struct.unpack("<q", h)
            recs.append(np.frombuffer(f.read(8 * cnt), dtype=np.float64))
    return recs


@pytest.mark.gpu
@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_dropin_matches_oracle(port, tmp_path, precision):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    n, dim, chunk, lq, bud, cfg, temp = 768, 128, 256, 64, (24, 40), (128, 384, 128), 0.9
    q, k, v = port.random_input(77, n, dim)
    q, k, v = (rounded(x, precision) for x in (q, k, v))
    inp = tmp_path / "in.bin"
    with open(inp, "wb") as f:
        f.write(struct.pack("<10q", n, dim, *cfg, chunk, lq, *bud, int(precision == "bf16")))
        f.write(struct.pack("<d", temp))
        for x in (q, k, v):
            f.write(np.ascontiguousarray(x, np.float64).tobytes())
    out = tmp_path / "out.bin"
    r = subprocess.run([build_binary(), str(inp), str(out)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    rec = iter(_read_records(out))
    tol = TOL[precision]
    # 1. chunked_prefill (sparse, DcaContinuous)
    o_ref, l_ref, sels = port.chunked_prefill(q, k, v, chunk, lq, bud, "sparse", 1, cfg,
                                              temperature=temp)
    o, lse = next(rec).reshape(n, dim), next(rec)
    assert int(next(rec)[0]) == len(sels)
    for s in sels:
        assert next(rec).astype(int).tolist() == s.critical.verticals
        assert next(rec).astype(int).tolist() == s.critical.slashes
    assert row_rel_err(o, o_ref) <= tol and lse_rel_err(lse, l_ref) <= tol
    # 2. estimate_block -> select_critical (on the device's fp32 scores) -> sparse_attention
    est = next(rec).reshape(min(lq, n), n)
    assert row_rel_err(est, port.estimate_block(q, k, lq)) <= 1e-5
    crit = port.select_critical(est.astype(np.float32).astype(np.float64), bud, n)
    assert next(rec).astype(int).tolist() == crit.verticals
    assert next(rec).astype(int).tolist() == crit.slashes
    o_ref, l_ref = port.sparse_attention(q, k, v, crit, temperature=temp)
    o, lse = next(rec).reshape(n, dim), next(rec)
    assert row_rel_err(o, o_ref) <= tol and lse_rel_err(lse, l_ref) <= tol
    # 3. dense, DCA dense (fused remap), explicit rel-matrix override
    o_ref, l_ref = port.full_attention(q, k, v, temperature=temp)
    o, lse = next(rec).reshape(n, dim), next(rec)
    assert row_rel_err(o, o_ref) <= tol and lse_rel_err(lse, l_ref) <= tol
    o_ref, l_ref = port.dca_attention(q, k, v, cfg, 2.0)
    o_dca, lse = next(rec).reshape(n, dim), next(rec)
    assert row_rel_err(o_dca, o_ref) <= tol and lse_rel_err(lse, l_ref) <= tol
    o_rel = next(rec).reshape(n, dim)
    assert row_rel_err(o_rel, o_ref) <= 1e-5
    # 3b. sparse attention under the RelPositionMatrix override (CUDA-core path)
    t_yarn = port.yarn_temperature(2.0)
    for c in (crit, Critical([5], [3], n)):
        o_ref, l_ref = port.sparse_attention(q, k, v, c, temperature=t_yarn, dca=cfg)
        o, lse = next(rec).reshape(n, dim), next(rec)
        assert row_rel_err(o, o_ref) <= TOL["fp32"] and lse_rel_err(lse, l_ref) <= TOL["fp32"]
    # 4. measure_budget_recall
    got = next(rec)[0]
    assert 0.0 < got <= 1.0
