"""Where does the host-entry time go? (GPU tool)"""
import sys
import time

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
od = torch.empty((n, 28, 128), dtype=torch.float32, device="cuda")


def t(fn, reps=2):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


print("h2d q+k+v ms", t(lambda: (q.copy_(qh, non_blocking=True), k.copy_(kh, non_blocking=True),
                                  v.copy_(vh, non_blocking=True))))
print("d2h out ms", t(lambda: oh.copy_(od, non_blocking=True)))
for prof in (False, True):
    context(0).set_profiling(prof)
    print("device prefill ms (profiling=%s)" % prof, t(lambda: D.chunked_prefill(q, k, v, **kw)))
    print("host entry ms (profiling=%s)" % prof,
          t(lambda: D.chunked_prefill_host(qh, kh, vh, out=oh, lse=lh, return_selections=True,
                                           **kw)))
context(0).set_profiling(False)
side = torch.cuda.Stream()


def overlap(copy):
    def run():
        with torch.cuda.stream(side):
            copy()
        D.chunked_prefill(q, k, v, **kw)
    return run


print("prefill + concurrent d2h ms", t(overlap(lambda: oh.copy_(od, non_blocking=True))))
q2 = torch.empty_like(q)
print("prefill + concurrent h2d ms", t(overlap(lambda: q2.copy_(qh, non_blocking=True))))
