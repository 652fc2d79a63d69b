"""Dump the tcgen05 pipeline trace of one chunked prefill (CTA 0, last chunk launch)."""
import ctypes as C
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2501_15383_b200 import device as D  # noqa: E402
from paper_2501_15383_b200._lib import context, lib  # noqa: E402
from paper_2501_15383_b200.synth import make_qkv, yarn_temperature  # noqa: E402
n, bv, bs = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
kind = sys.argv[4] if len(sys.argv) > 4 else "planted"
ctx = context(0)
L = lib()
L.lcx_debug_trace.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
L.lcx_debug_trace(ctx.ptr, 1, None)
q, k, v = make_qkv(n, 28, 4, kind=kind, seed=1)
s, c = 131072, 262144
D.chunked_prefill(q, k, v, chunk_len=32768, last_q=64, budget=(bv, bs),
                  position_mode="dca_continuous", dca=(s, c, min(s, c - s)),
                  temperature=yarn_temperature(n / c), rope_base=1e7)
buf = np.zeros((512, 8), np.int64)
L.lcx_debug_trace(ctx.ptr, 1, buf.ctypes.data)
t0 = buf[0, 0]
names = ["meta", "kTMA", "vTMA", "QKend", "PVend", "S_got", "P_put", "QKstart"]
print("tile " + " ".join(f"{x:>8s}" for x in names))
for t in range(0, 512, 1):
    row = buf[t]
    if row[0] == 0:
        break
    if t < 12 or (200 <= t < 216):
        print(f"{t:4d} " + " ".join(f"{(x - t0):8d}" for x in row[:8]))
d = np.diff(buf[:, 3][buf[:, 3] > 0])
print("median QK issue interval (clk):", np.median(d))
for c_, nm in [(0, "meta"), (1, "kTMA"), (5, "S_got"), (6, "P_put"), (4, "PV")]:
    x = buf[:, c_][buf[:, c_] > 0]
    print(nm, "median interval", np.median(np.diff(x)))
# latencies
m = (buf[:, 3] > 0) & (buf[:, 5] > 0)
print("QK issue -> softmax got S (median clk):", np.median((buf[:, 5] - buf[:, 3])[m]))
m = (buf[:, 6] > 0) & (buf[:, 5] > 0)
print("softmax got S -> P written (median clk):", np.median((buf[:, 6] - buf[:, 5])[m]))
m = (buf[:, 1] > 0) & (buf[:, 3] > 0)
print("K TMA issued -> QK issued (median clk):", np.median((buf[:, 3] - buf[:, 1])[m]))
m = (buf[:, 0] > 0) & (buf[:, 1] > 0)
print("meta ready -> K TMA issued (median):", np.median((buf[:, 1] - buf[:, 0])[m]))
m = (buf[:, 7] > 0) & (buf[:, 3] > 0)
print("QK issue duration (median):", np.median((buf[:, 3] - buf[:, 7])[m]))
pv = buf[:-1, 4]; top = buf[1:, 7]
m = (pv > 0) & (top > 0)
print("PV(t) issued -> MMA top(t+1) (median):", np.median((top - pv)[m]))
m = (buf[:, 6] > 0) & (buf[:, 4] > 0)
print("P_put(t) -> PV(t) issued (median):", np.median((buf[:, 4] - buf[:, 6])[m]))
m = (buf[:, 2] > 0) & (buf[:, 4] > 0)
print("vTMA(t) issued -> PV(t) issued (median):", np.median((buf[:, 4] - buf[:, 2])[m]))
a = buf[4:, 2]; b = buf[:-4, 4]; m = (a > 0) & (b > 0)
print("PV(t-4) issued -> vTMA(t) issued (median):", np.median((a - b)[m]))
a = buf[4:, 7]; b = buf[:-4, 4]; m = (a > 0) & (b > 0)
print("PV(t-4) issued -> QK(t) start (median):", np.median((a - b)[m]))
