"""Why the attention kernel's QK^T runs three MMA products (bf16 hi/lo split) and not one:
output error of causal attention on bf16-stored Q/K/V (Qwen2.5 head dim 128, rope base 1e7,
YaRN t(4)) when the fp32-rotated, scaled q and k are rounded to one fp16 / bf16 term, vs the
3-term split the kernel uses, against fp64 -- per-row max |o - o_ref| / max |o_ref| (the
2e-3 bf16 contract).  CPU only:  python tools/qk_precision.py [planted|iid]
"""
import math
import sys

import numpy as np
import torch

torch.manual_seed(0)
n, D = 2048, 128
kind = sys.argv[1] if len(sys.argv) > 1 else "planted"
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_2501_15383_b200 import synth
q, k, v = synth.make_qkv(n, 1, 1, D, kind=kind, device="cpu", rope_base=1e7)
q = q[:, 0].double().numpy(); k = k[:, 0].double().numpy(); v = v[:, 0].double().numpy()
th = np.array([1e7 ** (-2.0 * p / D) for p in range(D // 2)])
def rope(x, pos):
    a = pos[:, None] * th[None, :]
    c, s = np.cos(a), np.sin(a)
    xa, xb = x[:, 0::2], x[:, 1::2]
    out = np.empty_like(x); out[:, 0::2] = xa * c - xb * s; out[:, 1::2] = xa * s + xb * c
    return out
pos = np.arange(n, dtype=np.float64)
t = 1.0 / (0.1 * math.log(4) + 1) ** 2
scale = 1.0 / (t * math.sqrt(D))
qr, kr = rope(q, pos) * scale, rope(k, pos)
S = qr @ kr.T
mask = np.tril(np.ones((n, n), bool))
def attn(S):
    S = np.where(mask, S, -np.inf)
    m = S.max(1, keepdims=True); p = np.exp(S - m); return (p / p.sum(1, keepdims=True)) @ v
ref = attn(S)
def f16(x): return x.astype(np.float32).astype(np.float16).astype(np.float64)
def bf(x): return torch.tensor(x).to(torch.bfloat16).double().numpy()
def err(o): return (np.abs(o - ref).max(1) / np.abs(ref).max(1))
for name, S2 in [("f16x1", f16(qr.astype(np.float32)) @ f16(kr.astype(np.float32)).T),
                 ("bf16x1", bf(qr) @ bf(kr).T),
                 ("f16 q2 k1", qr @ f16(kr).T),
                 ("bf16 3-term", (lambda qh, kh: qh @ kh.T + qh @ bf(kr - kh).T + bf(qr - qh) @ kh.T)(bf(qr), bf(kr)))]:
    e = err(attn(S2.astype(np.float32).astype(np.float64)))
    print(name, "max %.2e  p99.9 %.2e mean %.2e" % (e.max(), np.quantile(e, 0.999), e.mean()))
