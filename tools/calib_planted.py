"""Calibrate the planted generator at scale: recall, slash locality and time (GPU tool)."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2501_15383_b200 import device as D  # noqa: E402
from paper_2501_15383_b200.synth import make_planted, yarn_temperature  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
s, c = 131072, 262144
kw = dict(chunk_len=32768, last_q=64, position_mode="dca_continuous", dca=(s, c, s),
          temperature=yarn_temperature(n / c), rope_base=1e7)
for local, band, anchor, heavy in [(10.6, 4096, 4.0, 28.0), (8.0, 4096, 4.0, 28.0),
                                   (12.0, 2048, 4.0, 28.0), (10.6, 16384, 4.0, 28.0)]:
    q, k, v = make_planted(n, 28, 4, local=local, band=band, anchor=anchor, heavy=heavy, seed=1)
    for bud in [(1000, 6096), (1000, 64)]:
        D.chunked_prefill(q, k, v, budget=bud, **kw)
        torch.cuda.synchronize()
        t0 = time.time()
        r = D.chunked_prefill(q, k, v, budget=bud, return_recall=True, return_admitted=True,
                              **kw)
        torch.cuda.synchronize()
        wall = time.time() - t0
        sl = r["slashes"].float()
        print(json.dumps(dict(local=local, band=band, anchor=anchor, heavy=heavy, budget=bud,
                              wall_s=round(wall, 3), tok_s=round(n / wall),
                              recall_mean=float(r["recall"].mean()),
                              recall_min=float(r["recall"].min()),
                              E=int(r["admitted"].sum()),
                              frac_slash_lt_8k=float((sl < 8192).float().mean()))), flush=True)
    del q, k, v
    torch.cuda.empty_cache()
