"""tc_min (entries of a 64-key slash tile for it to go to the tensor cores instead of the
CUDA-core gather) sweep at 1M tokens, 7B heads, budget (1000, 6096), per input kind:
device ms per layer and the attention stage split.  python tools/sweep_tcmin.py [kinds...]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_15383_b200 import device as D  # noqa: E402
from paper_2501_15383_b200._lib import context  # noqa: E402
from paper_2501_15383_b200.synth import make_qkv, yarn_temperature  # noqa: E402

n = 1 << 20
kinds = sys.argv[1:] or ["planted", "structured", "iid"]
s, c = 131072, 262144
kw = dict(chunk_len=32768, last_q=64, budget=(1000, 6096), position_mode="dca_continuous",
          dca=(s, c, min(s, c - s)), temperature=yarn_temperature(n / c), rope_base=1e7)
ctx = context(0)
ctx.set_profiling(True)
out = torch.empty((n, 28, 128), dtype=torch.float32, device="cuda")
lse = torch.empty((28, n), dtype=torch.float32, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for kind in kinds:
    q, k, v = make_qkv(n, 28, 4, kind=kind, seed=1)
    grid = os.environ.get("TCMIN")
    for tcm in ([int(x) for x in grid.split(",")] if grid else
                [16, 32, 48, 64, 96, 128] if kind == "planted" else [32, 64, 96, 160, 256]):
        D.chunked_prefill(q, k, v, out=out, lse=lse, tc_min_entries=tcm, **kw)
        torch.cuda.synchronize()
        ev[0].record()
        D.chunked_prefill(q, k, v, out=out, lse=lse, tc_min_entries=tcm, **kw)
        ev[1].record()
        torch.cuda.synchronize()
        st = ctx.stats()
        print(json.dumps(dict(kind=kind, tc_min=tcm, ms=ev[0].elapsed_time(ev[1]),
                              attn_tc=st["ms_tc_kernel"],
                              gather=st["ms_attention"] - st["ms_tc_kernel"],
                              gather_entries=st["simt_entries"])), flush=True)
    del q, k, v
