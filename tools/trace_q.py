"""Per-quadrant-warp softmax timeline of CTA 0 (build with
LCX_NVCC_EXTRA='-DLCX_TC_TRACE -DLCX_TC_TRACE_SM -DLCX_TC_TRACE_Q'): for each tile, when each of
the owner group's four quadrant warps got S and put P."""
import ctypes as C
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_2501_15383_b200 import device as D  # noqa: E402
from paper_2501_15383_b200._lib import context, lib  # noqa: E402
from paper_2501_15383_b200.synth import make_qkv, yarn_temperature  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1048576
ctx = context(0)
L = lib()
L.lcx_debug_trace.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
L.lcx_debug_trace(ctx.ptr, 1, None)
q, k, v = make_qkv(n, 28, 4, kind="planted", seed=1)
s, c = 131072, 262144
D.chunked_prefill(q, k, v, chunk_len=32768, last_q=64, budget=(1000, 6096),
                  position_mode="dca_continuous", dca=(s, c, min(s, c - s)),
                  temperature=yarn_temperature(n / c), rope_base=1e7)
buf = np.zeros((512 * 8 + 64,), np.int64)
L.lcx_debug_trace(ctx.ptr, 1, buf.ctypes.data)
buf = buf[:4096].reshape(512, 8)
t0 = buf[1, 0] if (len(sys.argv) > 2 and sys.argv[2] == 'meta') else buf[1, 4]
mode2 = len(sys.argv) > 2 and sys.argv[2] == "meta"
print("tile grp   " + ("meta start (wq0..3) | meta phase clk (wq0..3)" if mode2 else
                      "S_got(wq0..3)                  P_put(wq0..3)"))
for t in range(1, 400):
    b = buf[t]
    if b[4] == 0:
        break
    if mode2:
        print(f"{t:4d} {t & 1:3d} " + " ".join(f"{(x - t0):7d}" for x in b[0:4]) + "  |"
              + " ".join(f"{(y - x):6d}" for x, y in zip(b[0:4], b[4:8])))
        continue
    print(f"{t:4d} {t & 1:3d} " + " ".join(f"{(x - t0):7d}" for x in b[4:8]) + "  |"
          + " ".join(f"{(x - t0):7d}" for x in b[0:4]))
