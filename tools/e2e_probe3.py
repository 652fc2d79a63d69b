import sys, time
import torch
sys.path.insert(0, ".")
from paper_2501_15383_b200 import device as D  # noqa: E402
from paper_2501_15383_b200._lib import context  # noqa: E402
from paper_2501_15383_b200.synth import make_qkv, yarn_temperature  # noqa: E402
n = 1 << 20
q, k, v = make_qkv(n, 28, 4, seed=1)
s, c = 131072, 262144
kw = dict(chunk_len=32768, last_q=64, budget=(1000, 6096), position_mode="dca_continuous",
          dca=(s, c, s), temperature=yarn_temperature(n / c), rope_base=1e7)
qh, kh, vh = (torch.empty(x.shape, dtype=x.dtype, pin_memory=True) for x in (q, k, v))
qh.copy_(q); kh.copy_(k); vh.copy_(v)
oh = torch.empty((n, 28, 128), dtype=torch.float32, pin_memory=True)
lh = torch.empty((28, n), dtype=torch.float32, pin_memory=True)
for prof in (True, False, True, False):
    context(0).set_profiling(prof)
    for sel in (True, False):
        ts = []
        for rep in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            D.chunked_prefill_host(qh, kh, vh, out=oh, lse=lh, return_selections=sel, **kw)
            ts.append((time.perf_counter() - t0) * 1e3)
        print("profiling", prof, "selections", sel, [round(x) for x in ts], flush=True)
