"""Config C4 (BASELINE.json configs[3]): sparsity-refinement recall vs the (V, S) budget at
256K tokens, Qwen2.5-7B heads, DCA, with the operator's built-in recall check (dense vs
sparse LSE of every chunk's last 64 rows).  Prints one JSON line per budget.

    python tools/recall_sweep.py [n] [kind]
"""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2501_15383_b200 import device as D  # noqa: E402
from paper_2501_15383_b200.synth import make_qkv, yarn_temperature  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
kind = sys.argv[2] if len(sys.argv) > 2 else "planted"
q, k, v = make_qkv(n, 28, 4, kind=kind, seed=1)
s, c = 131072, 262144
kw = dict(chunk_len=32768, last_q=64, position_mode="dca_continuous", dca=(s, c, s),
          temperature=yarn_temperature(n / c), rope_base=1e7)
for bv in (64, 256, 1024, 4096):
    for bs in (64, 256, 1024, 4096):
        D.chunked_prefill(q, k, v, budget=(bv, bs), **kw)  # warm
        torch.cuda.synchronize()
        t0 = time.time()
        r = D.chunked_prefill(q, k, v, budget=(bv, bs), return_recall=True,
                              return_admitted=True, **kw)
        torch.cuda.synchronize()
        rec = r["recall"].float()
        E = int(r["admitted"].sum())
        print(json.dumps(dict(n=n, kind=kind, budget=[bv, bs], recall_mean=float(rec.mean()),
                              recall_min=float(rec.min()),
                              density=E / (28 * n * (n + 1) / 2), wall_s=time.time() - t0)),
              flush=True)
