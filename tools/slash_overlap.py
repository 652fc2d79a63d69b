"""How much do the heads of one GQA group share selected lines? (GPU tool, not a test)"""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2501_15383_b200 import device as D  # noqa: E402
from paper_2501_15383_b200.synth import make_qkv, yarn_temperature  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
kind = sys.argv[2] if len(sys.argv) > 2 else "structured"
q, k, v = make_qkv(n, 28, 4, kind=kind, seed=1)
s, c = 131072, 262144
r = D.chunked_prefill(q, k, v, chunk_len=32768, last_q=64, budget=(1000, 6096),
                      position_mode="dca_continuous", dca=(s, c, s), temperature=yarn_temperature(n / c),
                      rope_base=1e7)
V, NV, S, NS = (r[x].cpu() for x in ("verticals", "nv", "slashes", "ns"))
out = []
for ci in range(0, V.shape[0], max(1, V.shape[0] // 8)):
    for g in range(4):
        sl = [set(S[ci, h, :int(NS[ci, h])].tolist()) for h in range(g * 7, g * 7 + 7)]
        vl = [set(V[ci, h, :int(NV[ci, h])].tolist()) for h in range(g * 7, g * 7 + 7)]
        us, uv = set().union(*sl), set().union(*vl)
        out.append(dict(chunk=ci, g=g, slash_sum=sum(map(len, sl)), slash_union=len(us),
                        vert_sum=sum(map(len, vl)), vert_union=len(uv)))
for o in out:
    print(json.dumps(o))
