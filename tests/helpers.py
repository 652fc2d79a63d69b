"""Test helpers: precision rounding and the tolerance norms of DESIGN.md (D1)."""
import numpy as np


def rounded(x, precision):
    """Round a float64 array to the device storage type and back (what both sides see)."""
    import torch
    t = torch.as_tensor(np.asarray(x, dtype=np.float64))
    dt = torch.float32 if precision == "fp32" else torch.bfloat16
    return t.to(dt).to(torch.float64).numpy()


def row_rel_err(out, ref):
    """max over rows of max_d |o - o_ref| / max_d |o_ref|."""
    out, ref = np.asarray(out, np.float64), np.asarray(ref, np.float64)
    den = np.maximum(np.abs(ref).max(axis=-1), 1e-30)
    return float((np.abs(out - ref).max(axis=-1) / den).max())


def lse_rel_err(lse, ref):
    lse, ref = np.asarray(lse, np.float64), np.asarray(ref, np.float64)
    return float((np.abs(lse - ref) / np.maximum(np.abs(ref), 1.0)).max())


TOL = {"fp32": 1e-5, "bf16": 2e-3}


def check_selection(port, got_v, got_s, col32, sl32, col64, sl64, t1, block, budget,
                    sink=True, band=True, rel=1e-5):
    """The index contract: (1) the device selection is identical to the reference ranking
    of the device's own fp32 scores (ties -> lowest index); (2) where it differs from the
    selection of the fp64 reference scores, the differing lines are near-ties: their fp64
    score lies within `rel` (relative to the largest score) of the selection threshold."""
    crit = port.select_from_scores(col32, sl32, t1, block, budget, sink, band)
    assert list(got_v) == crit.verticals, "verticals differ from the ranking of own scores"
    assert list(got_s) == crit.slashes, "slashes differ from the ranking of own scores"
    ref = port.select_from_scores(col64, sl64, t1, block, budget, sink, band)
    ties = []
    for kind, got, want, score, k in (("vertical", got_v, ref.verticals, col64, budget[0]),
                                      ("slash", got_s, ref.slashes, sl64, budget[1])):
        diff = set(got) ^ set(want)
        if not diff:
            continue
        finite = np.where(np.isfinite(score), score, -np.inf)
        thresh = np.sort(finite)[::-1][min(k, len(finite)) - 1]
        scale = np.abs(finite[np.isfinite(finite)]).max()
        for x in sorted(diff):
            margin = abs(score[x] - thresh) / scale
            ties.append({"line": kind, "index": int(x), "in_device": x in set(got),
                         "score64": float(score[x]), "threshold64": float(thresh),
                         "margin_rel_max": float(margin)})
            assert abs(score[x] - thresh) <= rel * scale, (x, score[x], thresh)
    return ties
