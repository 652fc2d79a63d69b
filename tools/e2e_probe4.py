"""Host entry vs device-resident prefill on the bench workload: wall times and the
per-stage device times of each (GPU tool)."""
import sys
import time
import torch
sys.path.insert(0, ".")
from paper_2501_15383_b200 import device as D  # noqa: E402
from paper_2501_15383_b200._lib import context  # noqa: E402
from paper_2501_15383_b200.synth import make_qkv, yarn_temperature  # noqa: E402
n = 1 << 20
q, k, v = make_qkv(n, 28, 4, kind="planted", seed=1)
s, c = 131072, 262144
kw = dict(chunk_len=32768, last_q=64, budget=(1000, 6096), position_mode="dca_continuous",
          dca=(s, c, s), temperature=yarn_temperature(n / c), rope_base=1e7)
qh, kh, vh = (torch.empty(x.shape, dtype=x.dtype, pin_memory=True) for x in (q, k, v))
qh.copy_(q); kh.copy_(k); vh.copy_(v)
oh = torch.empty((n, 28, 128), dtype=torch.float32, pin_memory=True)
lh = torch.empty((28, n), dtype=torch.float32, pin_memory=True)
ctx = context(0)


def run(name, fn, prof):
    ctx.set_profiling(prof)
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fn()
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3
    st = ctx.stats() if prof else {}
    keep = {k_: round(v_, 1) for k_, v_ in st.items() if k_.startswith("ms")}
    print(f"{name:28s} prof={prof} wall {ms:7.1f} ms {keep}", flush=True)


for prof in (False, True):
    run("device", lambda: D.chunked_prefill(q, k, v, **kw), prof)
    run("host sel", lambda: D.chunked_prefill_host(qh, kh, vh, out=oh, lse=lh,
                                                    return_selections=True, **kw), prof)
    run("host nosel", lambda: D.chunked_prefill_host(qh, kh, vh, out=oh, lse=lh,
                                                      return_selections=False, **kw), prof)
