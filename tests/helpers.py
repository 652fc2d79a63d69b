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
