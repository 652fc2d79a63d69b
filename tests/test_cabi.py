"""CPU checks of the drop-in boundary: the C-ABI library loads, exports every symbol
include/longctx_b200.h declares, and fails loudly (kind "cuda") without a GPU --
there is no CPU fallback.  No compute calls here."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "longctx_b200.h")


def declared_symbols():
    txt = open(HDR).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(lcx_\w+)\s*\(", txt, re.M)))


def test_header_declares_the_operator_set():
    syms = declared_symbols()
    for s in ["lcx_estimate_block", "lcx_line_scores", "lcx_select_from_scores",
              "lcx_select_critical", "lcx_sparse_attention", "lcx_full_attention",
              "lcx_chunked_prefill", "lcx_attention_recall", "lcx_lse_merge"]:
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_2501_15383_b200 import _lib
    L = _lib.lib()
    missing = [s for s in declared_symbols() if not hasattr(L, s)]
    assert not missing, missing
    assert set(_lib.EXPORTS) <= set(declared_symbols())


def test_library_is_sm100a_only():
    import subprocess
    from paper_2501_15383_b200 import _lib
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2501_15383_b200 import _lib
    with pytest.raises(_lib.Error) as e:
        _lib.Context(0)
    assert e.value.kind == "cuda"
    from paper_2501_15383_b200 import longctx
    import numpy as np
    inp = longctx.AttentionInput(np.zeros((4, 8)), np.zeros((4, 8)), np.zeros((4, 8)))
    with pytest.raises(_lib.Error) as e:
        longctx.full_attention(inp)
    assert e.value.kind == "cuda"


def test_status_codes_match_reference_kinds():
    from paper_2501_15383_b200 import _lib
    assert _lib.KINDS[1] == "dimension" and _lib.KINDS[2] == "config"
    assert _lib.KINDS[3] == "domain" and _lib.KINDS[4] == "causality"
    assert _lib.KINDS[5] == "empty_row" and _lib.KINDS[6] == "empty_calibration"


def test_python_mirror_validates_like_the_reference():
    """Host-side validation errors (no device needed) carry the reference kinds."""
    import numpy as np
    from paper_2501_15383_b200 import longctx as L
    with pytest.raises(L.Error) as e:
        L.ChunkConfig(0, 4, 0).validate()
    assert e.value.kind == "config"
    with pytest.raises(L.Error) as e:
        L.ChunkConfig(6, 10, 5).validate()
    assert e.value.kind == "config"
    bad = L.AttentionInput(np.zeros((3, 8)), np.zeros((3, 8)), np.full((3, 8), np.nan))
    with pytest.raises(L.Error) as e:
        bad.validate()
    assert e.value.kind == "domain"
    odd = L.AttentionInput(np.zeros((3, 7)), np.zeros((3, 7)), np.zeros((3, 7)))
    with pytest.raises(L.Error) as e:
        odd.validate()
    assert e.value.kind == "config"
    with pytest.raises(L.Error) as e:
        L.selection_position(0, 1, L.ChunkConfig(6, 10, 4))
    assert e.value.kind == "causality"
    assert L.selection_position(7, 5, L.ChunkConfig(6, 10, 4)) == 2
    assert L.selection_position(13, 0, L.ChunkConfig(6, 10, 4)) == 9
    assert L.dca_relative(11, 2, L.ChunkConfig(6, 10, 4)) == 7
    assert abs(L.yarn_temperature(4.0) - 0.771321) < 1e-6
    crit = L.CriticalSet([5], [], 8)
    assert crit.admitted_row(2) == [2] and crit.admitted_row(6) == [5]
    assert crit.admitted_count() == 5 + 3
