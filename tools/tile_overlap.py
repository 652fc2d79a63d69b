"""Fraction of tensor-core slash tiles (relative 64-key tiles with >= 96 entries) shared by
the query heads of one KV head (GPU tool, not a test)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2501_15383_b200 import device as D  # noqa: E402
from paper_2501_15383_b200.synth import make_qkv, yarn_temperature  # noqa: E402

n = 1 << 20
q, k, v = make_qkv(n, 28, 4, kind="structured", seed=1)
s, c = 131072, 262144
r = D.chunked_prefill(q, k, v, chunk_len=32768, last_q=64, budget=(1000, 6096),
                      position_mode="dca_continuous", dca=(s, c, s),
                      temperature=yarn_temperature(n / c), rope_base=1e7)
S, NS = r["slashes"].cpu().numpy(), r["ns"].cpu().numpy()


def tiles(ds):
    hist = {}
    for d in ds:
        u_lo = -((d + 63) >> 6) - 1
        for u in range(u_lo, min(u_lo + 5, 2)):
            r0, r1 = max(0, d + 64 * u), min(128, d + 64 * u + 64)
            if r1 > r0:
                hist[u] = hist.get(u, 0) + r1 - r0
    return {u for u, x in hist.items() if x >= 96}


for ci in (8, 16, 24, 31):
    for g in range(4):
        ts = [tiles(S[ci, h, :NS[ci, h]].tolist()) for h in range(7 * g, 7 * g + 7)]
        tot = sum(map(len, ts))
        uni = len(set().union(*ts))
        print(json.dumps(dict(chunk=ci, g=g, tc_tiles_sum=tot, union=uni,
                              reuse=round(tot / max(uni, 1), 2))))
