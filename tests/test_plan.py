"""Sparsity plans, their JSON, and budget refinement through
the C++ drop-in (tests/cpp/plan_parity.cpp), against fixtures the reference produced
(tests/golden/make_refine_golden.py), plus DCPP chunk sizing (§8(f) row 4):

  * CPU: CriticalSet / SparsityPlan / prefill-selection JSON text equals what the
    reference CLI wrote (proj/out/sparsity/critical_set.json, prefill_selections.json,
    proj/out/refine/plan_refined.json), round trips,
    and malformed plans / configs raise the reference's error kinds;
  * GPU: refine_plan and offline_search reproduce the reference's budgets, rounds and
    plans exactly and its recalls within 1e-4, on the reference's refinement scenarios
    (planted columns that need growth, converged heads, a diffuse head at the cap,
    several heads and samples, FractionAbove, an offline grid).
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "plan_parity.cpp")
BIN = os.path.join(ROOT, "tests", "cpp", "plan_parity")
GOLD = os.path.join(ROOT, "tests", "golden")


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


def test_plan_json_matches_reference_text():
    r = subprocess.run([build_binary(), "--json", os.path.join(GOLD, "ref_critical_set.json"),
                        os.path.join(GOLD, "ref_plan_refined.json"),
                        os.path.join(GOLD, "ref_prefill_selections.json")],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


def test_dcpp_schedules_match_reference():
    r = subprocess.run([build_binary(), "--dcpp", os.path.join(GOLD, "dcpp_golden.txt")],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_measured_chunk_costs_feed_dcpp():
    r = subprocess.run([build_binary(), "--measure"], capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_refine_and_offline_search_match_reference():
    r = subprocess.run([build_binary(), "--refine", os.path.join(GOLD, "refine_golden.txt")],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "refine cases: 6" in r.stdout, r.stdout
